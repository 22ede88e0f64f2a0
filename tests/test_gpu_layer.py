"""GPU parity of the whole TP layer step (attention-projection block + MLP
block, fwd + bwd) through the C ABI against the oracle's layer_step, on the
same seeded inputs: ZERO-resizing at several ratios, Zero imputation, the
producer-side compaction path, and SEMI migration (hidden units appended on
helpers).  Multi-rank runs are simulated on one GPU with one context per rank;
the test itself sums the partials where NCCL would (test plumbing only)."""
import math

import numpy as np
import pytest

from oracle import ztp_oracle as O
from synth import inputs as I

pytestmark = pytest.mark.gpu
TOL = 2e-2


def make_inputs(h, f, N, e, seed):
    Wq, Wk, Wv, Wo = (I.uniform_sym(seed, n, h, h, 1 / math.sqrt(h)) for n in ("wq", "wk", "wv", "wo"))
    W1 = I.uniform_sym(seed, "w1", h, f, 1 / math.sqrt(h))
    W2 = I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f))
    X = I.normal(seed, "x", h, N)
    G = I.normal(seed, "g", h, N)
    return X, G, O.shard_layer(Wq, Wk, Wv, Wo, W1, W2, e)


def to_dev(torch, a, dtype=None):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda().to(dtype or torch.bfloat16)


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def close(got, ref, name, tol=TOL):
    sc = max(np.max(np.abs(ref)), 1e-30)
    err = np.max(np.abs(got - ref)) / sc
    assert np.isfinite(got).all() and err <= tol, f"{name}: max|err|/||ref||inf = {err:.3e}"


def selections(e, h, f, N, seed, gam, own_fc2=None):
    """Oracle-side selections from the same seeded scores the device gets."""
    a, u = h // e, f // e
    sel, scores, nps = [], [], []
    for r in range(e):
        lens = {"qkv": h, "o": a, "fc1": h, "fc2": (own_fc2[r] if own_fc2 else u)}
        d, sc, npr = {}, {}, {}
        for s, L in lens.items():
            sc[s] = I.lognormal_scores(seed, f"score.{s}", L, rank=r)
            npr[s] = min(int(math.floor(L * gam[r][s] + 0.5)), L - 1)
            d[s] = O.select(sc[s], npr[s])
        sel.append(d)
        scores.append(sc)
        nps.append(npr)
    return sel, scores, nps


@pytest.fixture(scope="module")
def tz():
    import torch
    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.layer import ZtpLayer, MigrationIO
    assert torch.cuda.is_available()
    return torch, Z, ZtpLayer, MigrationIO


def build(tz, sh, r, e, h, f, N, cap=0, dtype=None, plain=False, attn=None):
    torch, Z, ZtpLayer, _ = tz
    dtype = dtype or torch.bfloat16
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    d = lambda a: to_dev(torch, a, dtype)  # noqa: E731
    L = ZtpLayer(ctx, h, f, N, r, e, {"qkv": d(sh.qkv_t[r]), "o": d(sh.o_t[r]), "w1": d(sh.w1_t[r]),
                                      "w2": d(sh.w2_t[r])}, mig_cap=cap, dtype=dtype, plain=plain, attn=attn)
    return ctx, L


@pytest.mark.parametrize("h,f,N,g", [(256, 1024, 328, (0.5, 0.3, 0.5, 0.4)),
                                     (128, 512, 256, (0.0, 0.0, 0.0, 0.0)),
                                     (192, 768, 520, (0.9, 0.25, 0.1, 0.75))])
def test_layer_world1_real_context(tz, h, f, N, g):
    """TP = 1 through the real single-rank context (collectives are no-ops)."""
    torch, Z, ZtpLayer, _ = tz
    seed = 99 + h
    X, G, sh = make_inputs(h, f, N, 1, seed)
    gam = [dict(zip(("qkv", "o", "fc1", "fc2"), g))]
    sel, scores, nps = selections(1, h, f, N, seed, gam)
    ref = O.layer_step(X, G, sh, sel)
    ctx, L = build(tz, sh, 0, 1, h, f, N)
    L.set_selection(nps[0], {s: torch.from_numpy(v).cuda() for s, v in scores[0].items()})
    L.X.copy_(to_dev(torch, X))
    L.G.copy_(to_dev(torch, G))
    L.step(select=True)
    Z.ztp_sync(ctx)
    close(host(L.Y), ref["Y"], "Y")
    close(host(L.dX), ref["dX"], "dX")
    close(host(L.dqkv), ref["dWqkv"][0], "dWqkv")
    close(host(L.do), ref["dWo"][0], "dWo")
    close(host(L.dw1[:, :f]), ref["dW1"][0], "dW1")
    close(host(L.dw2[:f]), ref["dW2"][0], "dW2")
    for seg, t in (("qkv", L.dqkv), ("o", L.do), ("fc1", L.dw1), ("fc2", L.dw2)):
        P = sel[0][seg][1]
        if len(P):
            assert torch.all(t[torch.tensor(P, device="cuda")] == 0)          # Zero imputation
    # executed FLOPs accounting matches the oracle's audit
    assert L.method_flops() == pytest.approx(ref["flops"][0], rel=1e-12)
    Z.ztp_ctx_destroy(ctx)


def test_layer_cuda_graph_replay(tz):
    """The bench replays the step as a CUDA graph: the captured step (select +
    fwd + bwd through the C ABI) must reproduce the oracle on replay."""
    torch, Z, ZtpLayer, _ = tz
    h, f, N = 256, 1024, 264
    X, G, sh = make_inputs(h, f, N, 1, 5)
    gam = [dict(qkv=0.5, o=0.25, fc1=0.5, fc2=0.5)]
    sel, scores, nps = selections(1, h, f, N, 5, gam)
    ref = O.layer_step(X, G, sh, sel)
    ctx, L = build(tz, sh, 0, 1, h, f, N)
    L.set_selection(nps[0], {s: torch.from_numpy(v).cuda() for s, v in scores[0].items()})
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        L.X.copy_(to_dev(torch, X))
        L.G.copy_(to_dev(torch, G))
        L.step(s)                      # warm-up (sizes workspaces)
        L.Y.zero_()
        L.dX.zero_()
        L.capture(s)
        for _ in range(3):
            L.replay()
    torch.cuda.synchronize()
    close(host(L.Y), ref["Y"], "Y")
    close(host(L.dX), ref["dX"], "dX")
    close(host(L.dw1[:, :f]), ref["dW1"][0], "dW1")
    Z.ztp_ctx_destroy(ctx)


def _simulate(tz, e, h, f, N, gam, mig=None, seed=7, sampled=None, f32=False, plain=False, attn=None):
    """e ranks on one GPU; the test sums partials where NCCL all-reduces.
    sampled = k: full-size run checked on k token columns (Y, dX) against the
    oracle computed for those columns only (layer_step_sampled).
    f32: the verification mode (A-30) -- fp32 operands, SIMT FFMA GEMMs,
    fp32 sums -- checked at 1e-5 relative."""
    torch, Z, ZtpLayer, MigrationIO = tz
    dt = torch.float32 if f32 else torch.bfloat16
    tol = 1e-5 if f32 else TOL
    u = f // e
    X, G, sh = make_inputs(h, f, N, e, seed)
    mig = mig or []
    own = [u] * e
    inc = {r: [] for r in range(e)}
    for (s, r, lo, hi) in mig:
        own[s] = min(own[s], lo)
        inc[r].append((s, lo, hi))
    sel, scores, nps = selections(e, h, f, N, seed, gam, own_fc2=own)
    if sampled:
        cols = np.unique(np.concatenate([np.linspace(0, N - 1, sampled).astype(np.int64), [N - 1]]))
        ref = O.layer_step_sampled(X, G, sh, sel, cols, mig)
    else:
        core = O.AttnCore(attn.head_dim, attn.seq, attn.causal) if attn is not None else None
        ref = O.layer_step(X, G, sh, sel, mig, core=core)
    cap = max([sum(hi - lo for (_, lo, hi) in inc[r]) for r in range(e)] + [0])
    ranks = [build(tz, sh, r, e, h, f, N, cap, dt, plain, attn) for r in range(e)]
    offs = {}
    for r, (ctx, L) in enumerate(ranks):
        off = 0
        for (s, lo, hi) in inc[r]:
            offs[(s, r, lo)] = off
            off += hi - lo
        L.set_migration(MigrationIO(n_mig=u - own[r], inc=inc[r]))
        L.set_selection(nps[r], {s: torch.from_numpy(v).cuda() for s, v in scores[r].items()})
        L.X.copy_(to_dev(torch, X, dt))
        L.G.copy_(to_dev(torch, G, dt))
    # weight migration (ztp_migrate's job on a multi-GPU box)
    for (s, r, lo, hi) in mig:
        Ls, Lr = ranks[s][1], ranks[r][1]
        o = u + offs[(s, r, lo)]
        Lr.w1_t[:, o:o + hi - lo].copy_(Ls.w1_t[:, lo:hi])
        Lr.w2_t[o:o + hi - lo].copy_(Ls.w2_t[lo:hi])

    def allreduce(name):
        tot = sum(getattr(L, name).float() for _, L in ranks)     # rank order, fp32
        for _, L in ranks:
            getattr(L, name).copy_(tot.to(dt))
    for _, L in ranks:
        L.fwd_attn()
    allreduce("Y1")
    for _, L in ranks:
        L.fwd_mlp()
    allreduce("Y")
    for _, L in ranks:
        L.bwd_mlp()
    allreduce("dY1")
    for _, L in ranks:
        L.bwd_attn()
    allreduce("dX")
    for (s, r, lo, hi) in mig:     # dW slices back to the owner
        Ls, Lr = ranks[s][1], ranks[r][1]
        o = u + offs[(s, r, lo)]
        Ls.dw1[:, lo:hi].copy_(Lr.dw1[:, o:o + hi - lo])
        Ls.dw2[lo:hi].copy_(Lr.dw2[o:o + hi - lo])
    torch.cuda.synchronize()
    L0 = ranks[0][1]
    if sampled:
        ct = torch.tensor(cols, device="cuda")
        close(host(L0.Y[:, ct]), ref["Y"], "Y (sampled)")
        close(host(L0.dX[:, ct]), ref["dX"], "dX (sampled)")
        for r, (ctx, L) in enumerate(ranks):
            # Zero imputation of the straggler's dW rows, exact -- on its own
            # units (migrated units' dW comes back from helpers that contract
            # over their own kept rows, A-33)
            for seg, t in (("qkv", L.dqkv), ("o", L.do), ("fc1", L.dw1[:, :own[r]]), ("fc2", L.dw2)):
                P = sel[r][seg][1]
                if len(P):
                    assert torch.all(t[torch.tensor(P, device="cuda")] == 0), (r, seg)
            Z.ztp_ctx_destroy(ctx)
        return
    close(host(L0.Y), ref["Y"], "Y", tol)
    close(host(L0.dX), ref["dX"], "dX", tol)
    for r, (ctx, L) in enumerate(ranks):
        close(host(L.dqkv), ref["dWqkv"][r], f"dWqkv[{r}]", tol)
        close(host(L.do), ref["dWo"][r], f"dWo[{r}]", tol)
        close(host(L.dw1[:, :u]), ref["dW1"][r], f"dW1[{r}]", tol)
        close(host(L.dw2[:u]), ref["dW2"][r], f"dW2[{r}]", tol)
        assert L.method_flops() == pytest.approx(ref["flops"][r], rel=1e-12)
        Z.ztp_ctx_destroy(ctx)


@pytest.mark.parametrize("opts", [{"GROUP": 1}, {"GROUP": 2}, {"CONC": 0}, {"SQUAT_GUARD": 0}, {"A_EARLY": 0},
                                  {"PART": 0}, {"PART": 2}, {"AUX_WEIGHT": 2.5}, {"FLAGS": 1},
                                  {"DW_SHARE": 0.8}, {"DW_SHARE": 1.6}, {"SPLITK": 0},
                                  {"SPLITK": 0, "SPREAD_EPI": 1}, {"SPLITK": 0, "SPREAD_EPI": 1, "GROUP": 1},
                                  {"SPREAD_EPI": 1}, {"ZERO_GENERIC": 0},
                                  {"TAIL_HALVES": 0}, {"LATE_O_DW": 1}])
def test_layer_schedule_variants_graph(tz, opts):
    """The scheduling options (ztp_set_option: grouped or concurrent or
    serial dX / dW, the SM split weight -- it changes the dW split-K counts --,
    split-K off, the core's stream-order guard) change launch order and
    summation splits only: a captured step under each still matches the
    oracle."""
    torch, Z, ZtpLayer, _ = tz
    h, f, N = 512, 2048, 1032
    X, G, sh = make_inputs(h, f, N, 1, 17)
    gam = [dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)]
    sel, scores, nps = selections(1, h, f, N, 17, gam)
    ref = O.layer_step(X, G, sh, sel)
    ctx, L = build(tz, sh, 0, 1, h, f, N)
    for k, v in opts.items():
        if k == "LATE_O_DW":       # layer call order: O dW after the core on the side stream (dw_side)
            L.late_o_dw = bool(v)
            continue
        Z.ztp_set_option(ctx, getattr(Z, "OPT_" + k), v)
        assert Z.ztp_get_option(ctx, getattr(Z, "OPT_" + k)) == v
    L.set_selection(nps[0], {s: torch.from_numpy(v).cuda() for s, v in scores[0].items()})
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        L.X.copy_(to_dev(torch, X))
        L.G.copy_(to_dev(torch, G))
        L.step(s)
        L.Y.zero_()
        L.dX.zero_()
        L.dqkv.zero_()
        L.capture(s)
        for _ in range(2):
            L.replay()
    torch.cuda.synchronize()
    close(host(L.Y), ref["Y"], "Y")
    close(host(L.dX), ref["dX"], "dX")
    close(host(L.dqkv), ref["dWqkv"][0], "dWqkv")
    close(host(L.do), ref["dWo"][0], "dWo")
    close(host(L.dw1[:, :f]), ref["dW1"][0], "dW1")
    close(host(L.dw2[:f]), ref["dW2"][0], "dW2")
    Z.ztp_ctx_destroy(ctx)


def test_layer_tp2_straggler_resized(tz):
    """c1-like: TP=2, rank 1 resized at gamma = 0.25 (Zero imputation)."""
    g0 = dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0)
    g1 = dict(qkv=0.25, o=0.25, fc1=0.25, fc2=0.25)
    _simulate(tz, 2, 128, 512, 264, [g0, g1])


def test_layer_tp4_semi_migration(tz):
    """TP=4, straggler 3 sheds its tail units to helpers ranked by
    r' = (r - 3 + 4) % 4 and resizes the rest."""
    e, h, f = 4, 256, 1024
    u = f // e
    g = [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0) for _ in range(e)]
    g[3] = dict(qkv=0.5, o=0.5, fc1=0.3, fc2=0.3)
    n_mig = 96
    lo = u - n_mig
    mig = [(3, 0, lo, lo + 32), (3, 1, lo + 32, lo + 64), (3, 2, lo + 64, lo + 96)]
    _simulate(tz, e, h, f, 328, g, mig)


def test_layer_tp4_migration_receiver_resizes(tz):
    """Multi-straggler plan: a resize-group straggler (rank 1) also receives
    migrated units (A-22) and prunes them along K with its own S_c (A-33)."""
    e, h, f = 4, 128, 512
    u = f // e
    g = [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0) for _ in range(e)]
    g[1] = dict(qkv=0.25, o=0.25, fc1=0.4, fc2=0.25)
    mig = [(0, 1, u - 40, u - 16), (0, 2, u - 16, u - 8), (0, 3, u - 8, u)]
    _simulate(tz, e, h, f, 136, g, mig)


def test_layer_priority_epoch_next1(tz):
    """NEXT-1 at the layer level: two epochs of ZtpLayer.priority_epoch (column
    variation with carry-over, PriDiff ratio, selection) give the oracle's
    scores (1e-4), counts and index sets (bit-exact)."""
    torch, Z, ZtpLayer, _ = tz
    h, f, N = 128, 512, 264
    seed = 301
    X, G, sh = make_inputs(h, f, N, 1, seed)
    ctx, L = build(tz, sh, 0, 1, h, f, N)
    lens = {"qkv": h, "o": h, "fc1": h, "fc2": f}
    sc0 = {s: I.lognormal_scores(seed, f"score.{s}", n) for s, n in lens.items()}
    L.set_selection({s: 0 for s in lens}, {s: torch.from_numpy(v).cuda() for s, v in sc0.items()})
    ref_delta = {s: sc0[s].astype(np.float64) for s in lens}
    P_prev = {s: None for s in lens}
    theta, gamma_t = 2e-4, 0.4
    for epoch in range(2):
        prev = {s: t.clone() for s, t in L.weight_rows().items()}
        prev_h = {s: host(t) for s, t in prev.items()}
        # "training": perturb the weights; rows pruned last epoch stay unchanged
        for s, t in L.weight_rows().items():
            upd = to_dev(torch, I.normal(seed + epoch, f"upd.{s}", t.shape[0], t.shape[1]) * 1e-3 *
                         (1 + np.arange(t.shape[0])[:, None] % 7))
            if P_prev[s] is not None and len(P_prev[s]):
                upd[torch.tensor(P_prev[s], device="cuda")] = 0
            t.add_(upd)
        nps = L.priority_epoch(prev, gamma_t, theta)
        torch.cuda.synchronize()
        for s in lens:
            cur_h = host(L.weight_rows()[s])
            d = O.priority_update(ref_delta[s], cur_h, prev_h[s], P_prev[s])
            got = L._scores[sum(lens[t] for t in list(lens)[:list(lens).index(s)]):][:lens[s]].cpu().numpy()
            assert np.allclose(got, d, rtol=1e-4, atol=1e-12), s
            g = min(O.pridiff_gamma(got, theta, gamma_t), 0.9)
            npr = min(int(g * lens[s] + 0.5), lens[s] - 1)
            assert nps[s] == npr, s
            S, P = O.select(got, npr)
            assert np.array_equal(L.S[s].cpu().numpy(), S) and np.array_equal(L.P[s][:npr].cpu().numpy(), P), s
            ref_delta[s], P_prev[s] = got.astype(np.float64), P
    Z.ztp_ctx_destroy(ctx)


# ---------------------------------------------- BASELINE.json configs, full size

def _tail(u, n_mig, s, e):
    """SEMI ranges of straggler s: tail [u - n_mig, u) split over the other
    ranks in r' = (r - s + e) % e order, remainder to the lowest r' (A-28)."""
    recv = sorted((r for r in range(e) if r != s), key=lambda r: (r - s + e) % e)
    m, rem = divmod(n_mig, len(recv))
    out, lo = [], u - n_mig
    for i, r in enumerate(recv):
        k = m + (1 if i < rem else 0)
        if k:
            out.append((s, r, lo, lo + k))
        lo += k
    return out


def _zeros(e):
    return [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0) for _ in range(e)]


def test_config_c2_full_size_sampled(tz):
    """c2 (GPT-2 medium, N = 8192) at TP = 1, gamma = 0.5 on every linear --
    the bench workload -- Y and dX checked on sampled token columns."""
    _simulate(tz, 1, 1024, 4096, 8192, [dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)], seed=241, sampled=24)


def test_config_c3_full_size_all_outputs(tz):
    """c3 (ViT-L, 197 x 64 = 12608 tokens) at TP = 4, rank 3 resized at 0.5:
    every output of every rank (Y, dX, dWqkv, dWo, dW1, dW2) against the full
    fp64 oracle step."""
    g = _zeros(4)
    g[3] = dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)
    _simulate(tz, 4, 1024, 4096, 12608, g, seed=242)


def test_config_c4_full_size_semi_all_outputs(tz):
    """c4 (Llama-2-7B-shaped, h = 4096, f = 11008, N = 2048) at TP = 8, rank 5
    a 3x straggler: SEMI with beta = 0.25 -> 229 of its 1376 units migrate to
    the 7 helpers (33,33,33,33,33,32,32 in r' order) and the rest resizes at
    gamma_r = 0.6.  Every output of every rank, the helpers' returned dW
    slices included, against the full fp64 oracle step."""
    e, f = 8, 11008
    g = _zeros(e)
    g[5] = dict(qkv=0.6, o=0.6, fc1=0.6, fc2=0.6)
    _simulate(tz, e, 4096, f, 2048, g, mig=_tail(f // e, 229, 5, e), seed=243)


def test_config_c5_layer_full_size_all_outputs(tz):
    """c5 (GPT-13B-shaped layer, h = 5120, f = 20480, N = 2048) at TP = 8,
    rank 0 resized at 0.5 (one layer of the 4-layer stack): every output of
    every rank against the full fp64 oracle step (~1 min of host fp64)."""
    g = _zeros(8)
    g[0] = dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)
    _simulate(tz, 8, 5120, 20480, 2048, g, seed=244)


def test_config_c0_paper_shape_all_outputs(tz):
    """c0 (optional, the paper's ViT-1B layer: h = 2048, f = 8192, 65 x 64 =
    4160 tokens) at TP = 8, rank 7 a 4x straggler resized at 0.75: every
    output of every rank against the full fp64 oracle step."""
    g = _zeros(8)
    g[7] = dict(qkv=0.75, o=0.75, fc1=0.75, fc2=0.75)
    _simulate(tz, 8, 2048, 8192, 4160, g, seed=245)


def test_config_c1_exact_shape(tz):
    """c1 (single FFN-block config of BASELINE.json: h = 64, f = 256, seq 16 x
    batch 2 -> N = 32) at TP = 2, rank 1 slowed 2x -> T_avg ratio 0.25 on every
    linear (the config's stated ratio, S:363 closed form), full comparison."""
    g = _zeros(2)
    g[1] = dict(qkv=0.25, o=0.25, fc1=0.25, fc2=0.25)
    _simulate(tz, 2, 64, 256, 32, g, seed=240)


def test_config_c2_full_size_all_outputs(tz):
    """The bench workload (c2, N = 8192, TP = 1, gamma = 0.5) compared on EVERY
    output against the full fp64 oracle step: Y, dX and the four weight
    gradients (split-K dW reduce with the dW1 column spread of output
    pruning, A-35, at production shapes)."""
    _simulate(tz, 1, 1024, 4096, 8192, [dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)], seed=241)


def test_config_c4_tp1_all_outputs(tz):
    """c4's bench workload (h = 4096, f = 11008, N = 2048, TP = 1, gamma = 0.5)
    on EVERY output against the full fp64 oracle step: at these shapes the
    output-pruned dWqkv (V pruning, A-36) and dW1 (A-35) run unsplit, their
    compact columns spread by ztp_expand_cols."""
    _simulate(tz, 1, 4096, 11008, 2048, [dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)], seed=243)


@pytest.mark.parametrize("e,gam,mig", [
    (1, [dict(qkv=0.5, o=0.25, fc1=0.5, fc2=0.4)], None),
    (2, [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0), dict(qkv=0.25, o=0.5, fc1=0.3, fc2=0.25)], None),
    (4, [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0)] * 3 + [dict(qkv=0.5, o=0.5, fc1=0.3, fc2=0.3)],
     [(3, 0, 64, 96), (3, 1, 96, 112), (3, 2, 112, 128)]),
])
def test_layer_f32_verification_mode(tz, e, gam, mig):
    """north_star's fp32 verification mode for the whole layer: fp32 operands,
    SIMT FFMA GEMMs, fp32 all-reduce sums, every output (Y, dX, all dW,
    SEMI included) within 1e-5 of ||ref||inf of the fp64 oracle."""
    _simulate(tz, e, 128, 512, 136, gam, mig=mig, seed=77 + e, f32=True)


def test_layer_plain_bf16_matches_oracle(tz):
    """The plain arrangement (no producer-side compaction, no output pruning)
    in bf16 gives the same results as the compacted one (both vs the oracle)."""
    g = _zeros(2)
    g[1] = dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)
    _simulate(tz, 2, 128, 512, 264, g, seed=55, plain=True)


@pytest.mark.parametrize("e,causal,gam", [
    (1, True, [dict(qkv=0.5, o=0.5, fc1=0.5, fc2=0.5)]),
    (1, False, [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0)]),
    (2, True, [dict(qkv=0.0, o=0.0, fc1=0.0, fc2=0.0), dict(qkv=0.25, o=0.5, fc1=0.3, fc2=0.25)]),
])
def test_layer_real_attention_core(tz, e, causal, gam):
    """NEXT-4: the layer with the real attention core (ztp_transpose around
    cuDNN's fused attention; heads whole per rank) vs the oracle's fp64
    softmax attention -- Y, dX and every dW, resized ranks included."""
    from paper_2401_11469_b200.layer import AttnSpec
    _simulate(tz, e, 256, 1024, 256, gam, seed=90 + e, attn=AttnSpec(head_dim=64, seq=64, causal=causal))


def test_transpose_with_column_selection(tz):
    """ztp_transpose: dst[i, r] = src[r, cols[i]] exactly (bf16 moves bits)."""
    torch, Z, _, _ = tz
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    src = torch.randn(77, 304, device="cuda").bfloat16()[:, :300]     # rows padded to 16 bytes (TMA rule)
    cols = torch.tensor([299, 0, 5, 17, 150, 151, 64, 33], dtype=torch.int32, device="cuda")
    dst = torch.zeros(8, 80, device="cuda", dtype=torch.bfloat16)
    Z.ztp_transpose(ctx, src, dst[:, :77], cols)
    full = torch.zeros(300, 80, device="cuda", dtype=torch.bfloat16)
    Z.ztp_transpose(ctx, src, full[:, :77])
    Z.ztp_sync(ctx)
    assert torch.equal(dst[:, :77], src[:, cols.long()].t())
    assert torch.equal(full[:, :77], src.t()) and torch.all(full[:, 77:] == 0)
    Z.ztp_ctx_destroy(ctx)

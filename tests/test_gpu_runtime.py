"""GPU tests of the runtime side of the path through the C ABI: SEMI-migration
peer copies at world 1 (local-copy path of ztp_migrate, a8), straggler
emulation + statistics (a1: M_i from the GEMMs' own stamps, A-6, A-32), the
statistics all-gather at world 1, and the profiling counters."""
import math

import numpy as np
import pytest

from oracle import ztp_oracle as O
from synth import inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_2401_11469_b200 as Z
    assert torch.cuda.is_available(), "GPU tests need a B200"
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    yield Z, torch, ctx
    Z.ztp_ctx_destroy(ctx)


def padded(torch, r, c, dtype, fill):
    ld = (c + 7) // 8 * 8 + 8
    t = torch.full((r, ld), fill, device="cuda", dtype=dtype)
    return t[:, :c]


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_migrate_local_copies(env, dtype):
    """Sub-matrix copies src[r0:r0+nr, c0:c0+nc] -> dst[dr0:.., dc0:..] (the
    W1 column / W2 row slices SEMI moves, A-26), exact; untouched elements
    keep their value; zero-size transfers are no-ops."""
    Z, torch, ctx = env
    td = torch.bfloat16 if dtype == "bf16" else torch.float32
    src = padded(torch, 300, 264, td, 0.0)
    src.copy_(torch.from_numpy(I.normal(3, "m", 300, 264).astype(np.float32)).cuda().to(td))
    dst = padded(torch, 280, 200, td, -7.0)
    xs = [Z.xfer(src, dst, r0=5, c0=8, nr=40, nc=64, dr0=0, dc0=16),
          Z.xfer(src, dst, r0=100, c0=0, nr=120, nc=24, dr0=150, dc0=100),
          Z.xfer(src, dst, r0=0, c0=0, nr=0, nc=10, dr0=0, dc0=0)]
    Z.ztp_migrate(ctx, xs)
    Z.ztp_sync(ctx)
    s, d = src.float().cpu().numpy(), dst.float().cpu().numpy()
    want = np.full((280, 200), -7.0, dtype=np.float32)
    want[0:40, 16:80] = s[5:45, 8:72]
    want[150:270, 100:124] = s[100:220, 0:24]
    assert np.array_equal(d, want)


def test_migrate_errors(env):
    Z, torch, ctx = env
    a = torch.zeros(64, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Z.ZtpError) as e1:
        Z.ztp_migrate(ctx, [Z.xfer(a, a, nr=8, nc=8, src_rank=0, dst_rank=1)])      # rank outside world 1
    assert e1.value.name == "ZTP_EINVAL"
    with pytest.raises(Z.ZtpError) as e2:
        Z.ztp_migrate(ctx, [Z.xfer(a, a, r0=60, nr=8, nc=8)])                      # slice outside src
    assert e2.value.name == "ZTP_ESHAPE"


def _gemm_args(Z, torch, K, n, N):
    x = (torch.rand(K, N, device="cuda") - 0.5).to(torch.bfloat16)
    w = (torch.rand(K, n, device="cuda") - 0.5).to(torch.bfloat16)
    y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
    return Z.linear_args(x_t=x, w_t=w, y_t=y), (x, w, y)


def test_slowdown_emulation_and_statistics(env):
    """chi = 2 stretches every GEMM to twice its own duration (delay kernel on
    the GEMM's %globaltimer stamps, A-32) and M_i accumulates the stretched
    time (A-6): M(chi=2) / M(chi=1) ~ 2.  The all-gather at world 1 returns
    the rank's own (T, M)."""
    Z, torch, ctx = env
    a, keep = _gemm_args(Z, torch, 2048, 2048, 8192)
    for _ in range(100):                             # clocks out of the idle state first
        Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    Z.ztp_set_slowdown(ctx, 2.0)                     # load the delay kernel (lazy module loading)
    Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    Z.ztp_sync(ctx)
    res = {}
    for chi in (1.0, 2.0):
        Z.ztp_set_slowdown(ctx, chi)
        Z.ztp_set_stats(ctx, True)
        Z.ztp_read_gemm_ns(ctx)                      # reset
        for _ in range(10):
            Z.ztp_gemm(ctx, Z.KIND_FWD, a)
        res[chi] = Z.ztp_read_gemm_ns(ctx)
        Z.ztp_set_stats(ctx, False)
    Z.ztp_set_slowdown(ctx, 1.0)
    assert res[1.0] > 0
    assert 1.7 < res[2.0] / res[1.0] < 2.3, res
    T, M = Z.ztp_allgather_stats(ctx, 1.25, 0.75, 1)
    assert T == [1.25] and M == [0.75]
    with pytest.raises(Z.ZtpError):
        Z.ztp_set_slowdown(ctx, 0.5)                 # chi < 1 is not a slowdown


def test_profile_counters(env):
    """ztp_read_profile: GEMM launch count and algorithmic FLOPs exact; the
    kernel-stamp time is positive and within the event-bracketed time."""
    Z, torch, ctx = env
    K, n, N = 512, 1024, 4096
    a, keep = _gemm_args(Z, torch, K, n, N)
    Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    torch.cuda.synchronize()
    Z.ztp_read_profile(ctx)
    Z.ztp_set_profile(ctx, True)
    for _ in range(3):
        Z.ztp_gemm(ctx, Z.KIND_FWD, a)
    p = Z.ztp_read_profile(ctx)
    Z.ztp_set_profile(ctx, False)
    assert p["n_gemm"] == 3
    assert p["gemm_flops"] == pytest.approx(3 * 2.0 * K * n * N, rel=1e-12)
    assert 0 < p["gemm_kernel_ms"] <= p["gemm_ms"] * 1.05


def test_options_round_trip_and_errors():
    """ztp_set_option / ztp_get_option (include/ztp.h): values round-trip,
    bad values and unknown options are EINVAL and leave the option as it was."""
    import paper_2401_11469_b200 as Z
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    try:
        for opt, val in ((Z.OPT_CONC, 0), (Z.OPT_DW_SHARE, 1.5), (Z.OPT_SQUAT_GUARD, 0), (Z.OPT_GATHER4, 1),
                         (Z.OPT_SPLITK, 0), (Z.OPT_GROUP, 2), (Z.OPT_PEER_CTAS, 16), (Z.OPT_A_EARLY, 0),
                         (Z.OPT_PART, 0), (Z.OPT_AUX_WEIGHT, 2.0), (Z.OPT_FLAGS, 1),
                         (Z.OPT_SPREAD_EPI, 1), (Z.OPT_ZERO_GENERIC, 0),
                         (Z.OPT_TAIL_HALVES, 0)):
            Z.ztp_set_option(ctx, opt, val)
            assert Z.ztp_get_option(ctx, opt) == val
        for opt, bad in ((Z.OPT_DW_SHARE, 0.0), (Z.OPT_GROUP, 3), (Z.OPT_PEER_CTAS, 0), (Z.OPT_PART, 3),
                         (Z.OPT_AUX_WEIGHT, -1.0), (99, 1.0)):
            with pytest.raises(Z.ZtpError) as ei:
                Z.ztp_set_option(ctx, opt, bad)
            assert ei.value.name == "ZTP_EINVAL"
        assert Z.ztp_get_option(ctx, Z.OPT_GROUP) == 2
    finally:
        Z.ztp_ctx_destroy(ctx)


@pytest.mark.parametrize("early,flags", [(1, 0), (0, 0), (1, 1)])
def test_gemm_chain_a_early(early, flags):
    """A-operand prefetch before the PDL wait (ZTP_OPT_A_EARLY): a chain of
    FWD GEMMs where (2) reads the output of (1) as B with an untouched A
    (prefetched early), (3) takes (1)'s output -- two launches back -- as its
    A (prefetched early: (2) triggers its dependents only after its own
    wait), (4) takes (3)'s output as A (not prefetched: the predecessor
    writes it).  Eager results match a plain fp32 matmul; 20 graph replays
    reproduce them bit for bit (a stale early read would differ)."""
    import torch
    import paper_2401_11469_b200 as Z
    ctx = Z.ztp_ctx_create(0, 1, None, 0)
    try:
        Z.ztp_set_option(ctx, Z.OPT_A_EARLY, early)
        Z.ztp_set_option(ctx, Z.OPT_FLAGS, flags)   # (2) then waits on (1)'s tile-completion counters
        g = torch.Generator(device="cpu").manual_seed(5)
        rnd = lambda r, c, s=1.0: ((torch.rand(r, c, generator=g) - 0.5) * s).cuda().to(torch.bfloat16)  # noqa
        K, n, N = 768, 512, 1536
        X, W1, W2, B3, B4 = rnd(K, N), rnd(K, n, 0.1), rnd(n, n, 0.2), rnd(n, n), rnd(N, n, 0.1)
        Y1 = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
        Y2 = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
        Y3 = torch.empty(N, n, device="cuda", dtype=torch.bfloat16)
        Y4 = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
        L = Z.linear_args
        steps = [L(x_t=X, w_t=W1, y_t=Y1),        # Y1^T = W1^T' X^T          (A = W1)
                 L(x_t=Y1, w_t=W2, y_t=Y2),       # Y2 = W2' Y1                (A = W2, B = Y1)
                 L(x_t=B3, w_t=Y1, y_t=Y3),       # Y3 = Y1' B3                (A = Y1: two launches back)
                 L(x_t=B4, w_t=Y3, y_t=Y4)]       # Y4 = Y3' B4                (A = Y3: the predecessor's output)
        s = torch.cuda.Stream()

        def run():
            for a in steps:
                Z.ztp_gemm(ctx, Z.KIND_FWD, a, s)
        with torch.cuda.stream(s):
            run()
        torch.cuda.synchronize()
        f = lambda t: t.float().cpu()  # noqa: E731
        r1 = f(W1).t() @ f(X)
        r2 = f(W2).t() @ f(Y1)
        r3 = f(Y1).t() @ f(B3)
        r4 = f(Y3).t() @ f(B4)
        for got, ref in ((Y1, r1), (Y2, r2), (Y3, r3), (Y4, r4)):
            err = (f(got) - ref).abs().max().item()
            assert err <= 0.02 * ref.abs().max().item() + 1e-3, err
        eager = [t.clone() for t in (Y1, Y2, Y3, Y4)]
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            run()
        for _ in range(20):
            for t in (Y1, Y2, Y3, Y4):
                t.fill_(7.0)
            gr.replay()
            torch.cuda.synchronize()
            for t, e in zip((Y1, Y2, Y3, Y4), eager):
                assert torch.equal(t, e)
    finally:
        Z.ztp_ctx_destroy(ctx)

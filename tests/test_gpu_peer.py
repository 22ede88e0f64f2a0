"""The multi-rank data plane executed for real: `world` OS processes on the
one GPU, each with its own context, joined by the peer-memory transport
(symmetric windows mapped through CUDA IPC; include/ztp.h "Peer-memory data
plane").  Covers a7 (all-reduce of row FWD / col BWD, unpaired all-gather,
P:112-119), a1's statistics exchange and a8's one-sided migration
pulls, bit-exact where the result is a plain definition and
against the fp64 oracle for a whole SEMI layer step (SURVEY §8(c) tolerances).
Each rank is tests/peer_worker.py."""
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import ztp_oracle as O
from synth import inputs as I

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL = 2e-2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_ranks(world, case, tmp_path, env=None, timeout=600):
    port = _free_port()
    e = dict(os.environ, **(env or {}))
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "peer_worker.py"), str(r), str(world),
                               str(port), case, str(tmp_path)], env=e, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=timeout)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{outs[r][-3000:]}"
    return [dict(np.load(os.path.join(tmp_path, f"{case}_{r}.npz"))) for r in range(world)]


def bf16(x):
    import torch
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_collectives_bit_exact(tmp_path, world):
    _check_collectives(run_ranks(world, "collectives", tmp_path), world)


def _check_collectives(res, world):
    # all-reduce: sum of the ranks' partials in rank order in fp32, one RNE
    # rounding for bf16 (the oracle's left fold)
    for tag in ("bf16", "f32"):
        acc = np.zeros_like(res[0][f"part_{tag}"], dtype=np.float32)
        for r in range(world):
            acc = (acc + res[r][f"part_{tag}"].astype(np.float32)).astype(np.float32)
        want = bf16(acc) if tag == "bf16" else acc
        for r in range(world):
            assert np.array_equal(res[r][f"sum_{tag}"], want), (tag, r)
    # all-gather: block q of every rank = rank q's own block
    n = res[0]["gathered"].shape[0] // world
    blocks = [res[q]["gathered"][q * n:(q + 1) * n] for q in range(world)]
    for r in range(world):
        assert np.array_equal(res[r]["gathered"], np.concatenate(blocks)), r
    # the gathered column FWD is the unsplit dense product
    K, N, seed = 96, 136, 4242
    Wt = I.uniform_sym(seed, "wc", K, world * n, 0.1)
    Xt = I.normal(seed, "xc", K, N)
    ref = Wt.T @ Xt
    assert np.max(np.abs(res[0]["gathered"] - ref)) <= TOL * np.max(np.abs(ref))
    # statistics
    for r in range(world):
        assert list(res[r]["T"]) == [1.25 + q for q in range(world)]
        assert list(res[r]["M"]) == [0.5 * q + 0.125 for q in range(world)]
    # pulls: rank d's B[5:22, 16:16+nc] = rank s's A[3+s:20+s, 8:8+nc], s = d+1 mod world; rest untouched
    for d in range(world):
        s = (d + 1) % world
        nc = 40 + 8 * s
        want = np.zeros_like(res[d]["B"])
        want[5:22, 16:16 + nc] = res[s]["A"][3 + s:20 + s, 8:8 + nc]
        assert np.array_equal(res[d]["B"], want), d


@pytest.mark.parametrize("world,mig,gamma", [
    (2, "192,256", "0.5,0.25,0.3,0.3"),                  # one helper
    (4, "80,96,96,112,112,128", "0.25,0.5,0.4,0.2"),     # three helpers, r' order
])
def test_peer_layer_step_semi(tmp_path, world, mig, gamma):
    """A whole TP layer step (select + FWD + BWD) with a SEMI plan through the
    peer transport, eager and replayed as a CUDA graph: Y, dX and every
    rank's weight gradients in the owner's view match the oracle."""
    _check_layer_semi(tmp_path, world, mig, gamma)


def _check_layer_semi(tmp_path, world, mig, gamma, env=None):
    res = run_ranks(world, "layer", tmp_path, env=dict({"PEER_MIG": mig, "PEER_GAMMA": gamma}, **(env or {})))
    h, f, N, seed = 128, 512, 264, 31
    e = world
    a, u = h // e, f // e
    s = e - 1
    spec = [int(v) for v in mig.split(",")]
    migl = [(s, r, spec[2 * k], spec[2 * k + 1]) for k, r in enumerate(x for x in range(e) if x != s)]
    own = [u] * e
    own[s] = migl[0][2]
    Wq, Wk, Wv, Wo = (I.uniform_sym(seed, n, h, h, 1 / math.sqrt(h)) for n in ("wq", "wk", "wv", "wo"))
    W1 = I.uniform_sym(seed, "w1", h, f, 1 / math.sqrt(h))
    W2 = I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f))
    X, G = I.normal(seed, "x", h, N), I.normal(seed, "g", h, N)
    sh = O.shard_layer(Wq, Wk, Wv, Wo, W1, W2, e)
    sel = []
    for r in range(e):
        lens = {"qkv": h, "o": a, "fc1": h, "fc2": own[r]}
        d = {}
        for k, (sg, L) in enumerate(lens.items()):
            npr = int(res[r]["nprune"][k])
            d[sg] = O.select(I.lognormal_scores(seed, f"score.{sg}", L, rank=r), npr)
        sel.append(d)
    ref = O.layer_step(X, G, sh, sel, migl)

    def close(got, want, name):
        err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30)
        assert np.isfinite(got).all() and err <= TOL, f"{name}: {err:.3e}"
    for r in range(e):
        close(res[r]["Y"], ref["Y"], f"Y[{r}]")
        close(res[r]["dX"], ref["dX"], f"dX[{r}]")
        close(res[r]["Y_graph"], ref["Y"], f"Y graph[{r}]")
        close(res[r]["dX_graph"], ref["dX"], f"dX graph[{r}]")
        close(res[r]["dqkv"], ref["dWqkv"][r], f"dWqkv[{r}]")
        close(res[r]["do"], ref["dWo"][r], f"dWo[{r}]")
        close(res[r]["dw1"], ref["dW1"][r], f"dW1[{r}]")
        close(res[r]["dw2"], ref["dW2"][r], f"dW2[{r}]")
        close(res[r]["dw1_graph"], ref["dW1"][r], f"dW1 graph[{r}]")
        # every rank holds the identical all-reduced tensors
        assert np.array_equal(res[r]["Y"], res[0]["Y"]) and np.array_equal(res[r]["dX"], res[0]["dX"])
    # Zero imputation of the straggler's own pruned dW rows is exact (its
    # migrated units' columns of dW1 come back whole from the helpers)
    for sg, key, cols in (("qkv", "dqkv", None), ("o", "do", None), ("fc1", "dw1", own[s])):
        P = sel[s][sg][1]
        if len(P):
            assert np.all(res[s][key][np.asarray(P)][:, :cols] == 0), sg


@pytest.mark.parametrize("world,migr,k,mode", [
    (3, "2", 96, "tree"), (3, "2", 96, "p2p"),        # one migrating rank, two helpers
    (4, "1,3", 130, "tree"), (4, "1,3", 250, "p2p"),  # nu = 2, ragged helper ranges
])
def test_peer_kdim_migration_lossless(tmp_path, world, migr, k, mode):
    """NEXT-3, the paper-literal sending-collecting migration of a column
    linear: migrating ranks shed k contraction rows to the normal
    ranks; outputs, dX (helpers' rows merged into the all-reduce) and
    every rank's dW (returned slices) equal the unsplit linear (P:233
    loss-free), eager and graph-replayed, under both policies."""
    res = run_ranks(world, "kmig", tmp_path, env={"PEER_MIGRATORS": migr, "PEER_K": str(k), "PEER_MODE": mode})
    K, n, N, seed = 256, 64, 136, 77
    X = I.normal(seed, "x", K, N)
    W = I.uniform_sym(seed, "w", K, world * n, 0.1)
    G = I.normal(seed, "g", world * n, N)
    dX = O.fold([O.linear_bwd_dx(W[:, r * n:(r + 1) * n], G[r * n:(r + 1) * n]) for r in range(world)])

    def close(got, want, name):
        err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30)
        assert np.isfinite(got).all() and err <= TOL, f"{name}: {err:.3e}"
    for r in range(world):
        Wr, Gr = W[:, r * n:(r + 1) * n], G[r * n:(r + 1) * n]
        for sfx in ("", "_graph"):
            close(res[r]["Y" + sfx], O.linear_fwd(Wr, X), f"Y{sfx}[{r}]")
            close(res[r]["dX" + sfx], dX, f"dX{sfx}[{r}]")
            close(res[r]["dW" + sfx], O.linear_bwd_dw(X, Gr), f"dW{sfx}[{r}]")


# ------------------------------------------------ one rank per GPU (>= 2 GPUs)

def _gpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multidev_peer_collectives_bit_exact(tmp_path, world):
    """Rank r on cuda:r (NVLink P2P between GPUs): the library's peer
    transport -- two-shot all-reduce in rank order, all-gather, statistics,
    one-sided pulls -- bit-exact as in the one-GPU run.  Skipped below
    `world` GPUs (the driver's boxes have one)."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    res = run_ranks(world, "collectives", tmp_path, env={"PEER_MULTIDEV": "1", "PEER_TRANSPORT": "peer"})
    _check_collectives(res, world)


@pytest.mark.parametrize("world,mig,gamma", [
    (2, "192,256", "0.5,0.25,0.3,0.3"),
    (4, "80,96,96,112,112,128", "0.25,0.5,0.4,0.2"),
])
def test_multidev_nccl_layer_step_semi(tmp_path, world, mig, gamma):
    """The SEMI layer step of test_peer_layer_step_semi with one rank per GPU
    and an NCCL communicator (collectives over NVLink / NVSwitch), migration
    pulls through the window: every output against the oracle.  Skipped
    below `world` GPUs."""
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    _check_layer_semi(tmp_path, world, mig, gamma, env={"PEER_MULTIDEV": "1", "PEER_TRANSPORT": "nccl"})

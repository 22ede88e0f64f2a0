"""One rank of a multi-process run of the peer-memory data plane
(include/ztp.h "Peer-memory data plane"): launched by tests/test_gpu_peer.py
as `world` OS processes, all on cuda:0 (CUDA IPC between processes of one
device is the same code path as NVLink P2P between GPUs).  Test plumbing
only: the handles are exchanged over a gloo group, every result is written to
<out>/<case>_<rank>.npz and checked by the parent test against the oracle or
the plain definition.

usage: python tests/peer_worker.py RANK WORLD PORT CASE OUTDIR
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, world, port, case, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    import torch
    import torch.distributed as dist

    import paper_2401_11469_b200 as Z
    from paper_2401_11469_b200.layer import MigrationIO, ZtpLayer, sym_allocator
    from synth import inputs as I

    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    # PEER_MULTIDEV=1 (>= world GPUs): rank r on cuda:r with an NCCL communicator
    # (collectives and grouped send / recv over NVLink) and the window mapped
    # across devices (peer pulls over NVLink); default: every rank on cuda:0,
    # peer transport over CUDA IPC
    multidev = os.environ.get("PEER_MULTIDEV") == "1"
    device = rank if multidev else 0
    torch.cuda.set_device(device)
    uid = None
    if multidev:
        box = [Z.ztp_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    ctx = Z.ztp_ctx_create(rank, world, uid, device)      # no NCCL id -> peer transport
    sym_alloc = lambda r, c, dt=torch.bfloat16: Z.ztp_sym_alloc(ctx, r, c, dt, device)  # noqa: E731

    def open_window(nbytes):
        h = Z.ztp_window_create(ctx, nbytes)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        Z.ztp_window_open(ctx, hs)
        if multidev and os.environ.get("PEER_TRANSPORT", "nccl") == "peer":
            Z.ztp_set_transport(ctx, Z.TRANSPORT_PEER)   # the library's own peer kernels across GPUs

    res = {}
    dev = lambda a, dt=torch.bfloat16: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda().to(dt)  # noqa
    host = lambda t: t.float().cpu().numpy()  # noqa: E731
    if case == "collectives":
        open_window(64 << 20)
        K, n, N, seed = 96, 80, 136, 4242
        # row-parallel FWD: partial (skip_collective) then the all-reduced sum
        for dt, tag in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
            Wt = I.uniform_sym(seed, "w", world * K, n, 0.1, r0=rank * K, r1=(rank + 1) * K)
            Xt = I.normal(seed, "x", world * K, N, r0=rank * K, r1=(rank + 1) * K)
            w, x = dev(Wt, dt), dev(Xt, dt)
            y = sym_alloc(n, N, dt)
            a = Z.linear_args(x_t=x, w_t=w, y_t=y, skip_collective=1)
            Z.ztp_row_linear(ctx, Z.FWD, a)
            torch.cuda.synchronize()
            res[f"part_{tag}"] = host(y)
            a = Z.linear_args(x_t=x, w_t=w, y_t=y)
            Z.ztp_row_linear(ctx, Z.FWD, a)
            Z.ztp_sync(ctx)
            res[f"sum_{tag}"] = host(y)
        # unpaired column FWD (gather_output): my block, then the all-gathered tensor
        Wt = I.uniform_sym(seed, "wc", K, world * n, 0.1, c0=rank * n, c1=(rank + 1) * n)
        Xt = I.normal(seed, "xc", K, N)
        yfull = sym_alloc(world * n, N)
        a = Z.linear_args(x_t=dev(Xt), w_t=dev(Wt), y_t=yfull, gather_output=True)
        Z.ztp_col_linear(ctx, Z.FWD, a)
        Z.ztp_sync(ctx)
        res["gathered"] = host(yfull)
        # statistics exchange
        T, M = Z.ztp_allgather_stats(ctx, 1.25 + rank, 0.5 * rank + 0.125, world)
        res["T"], res["M"] = np.array(T), np.array(M)
        # one-sided pulls: every rank's window tensor A holds rank-coded values;
        # rank r pulls a slice of rank (r+1) % world into its own B
        A = sym_alloc(64, 96)
        B = sym_alloc(64, 96)
        A.copy_(dev(I.normal(seed, "a", 64, 96, rank=rank)))
        B.zero_()
        xs = []
        for d in range(world):
            s = (d + 1) % world
            xs.append(Z.xfer(A, B, r0=3 + s, c0=8, nr=17, nc=40 + 8 * s, dr0=5, dc0=16, src_rank=s, dst_rank=d))
        Z.ztp_migrate(ctx, xs)
        Z.ztp_barrier(ctx)
        Z.ztp_sync(ctx)
        res["A"], res["B"] = host(A), host(B)
    elif case == "layer":
        # TP = world layer step, SEMI plan: the last rank sheds its tail units
        # to the others (r' order) and resizes; peer all-reduces,
        # ztp_migrate pulls of W1^T / W2^T slices out and dW slices back
        h, f, N, seed = 128, 512, 264, 31
        e = world
        a_, u = h // e, f // e
        s = e - 1
        spec = [int(v) for v in os.environ["PEER_MIG"].split(",")]     # lo, hi per helper (flattened)
        mig = [(s, r, spec[2 * k], spec[2 * k + 1]) for k, r in enumerate(x for x in range(e) if x != s)]
        cap = max(hi - lo for (_, _, lo, hi) in mig)
        open_window(ZtpLayer.window_bytes(h, f, N, e, cap) + (1 << 20))
        bq = 1 / math.sqrt(h)
        F0, F1, U0, U1 = rank * a_, (rank + 1) * a_, rank * u, (rank + 1) * u
        qkv = np.concatenate([I.uniform_sym(seed, nm, h, h, bq, c0=F0, c1=F1) for nm in ("wq", "wk", "wv")], axis=1)
        shards = {"qkv": dev(qkv), "o": dev(I.uniform_sym(seed, "wo", h, h, bq, r0=F0, r1=F1)),
                  "w1": dev(I.uniform_sym(seed, "w1", h, f, bq, c0=U0, c1=U1)),
                  "w2": dev(I.uniform_sym(seed, "w2", f, h, 1 / math.sqrt(f), r0=U0, r1=U1))}
        L = ZtpLayer(ctx, h, f, N, rank, e, shards, mig_cap=cap, alloc=sym_allocator(ctx, device))
        own = u - (u - mig[0][2] if rank == s else 0)
        all_x, inc = [], []
        for (src, dst, lo, hi) in mig:
            all_x.append((src, dst, lo, hi, 0))
            if dst == rank:
                inc.append((src, lo, hi))
        L.set_migration(MigrationIO(n_mig=u - own, inc=inc, all_xfers=all_x,
                                    out=[(d, lo, hi) for (_, d, lo, hi) in mig] if rank == s else []))
        gam = [float(g) for g in os.environ["PEER_GAMMA"].split(",")]    # per segment, straggler only
        lens = {"qkv": h, "o": a_, "fc1": h, "fc2": own}
        nps = {sg: (min(int(math.floor(Ln * g + 0.5)), Ln - 1) if rank == s else 0)
               for (sg, Ln), g in zip(lens.items(), gam)}
        sc = {sg: torch.from_numpy(I.lognormal_scores(seed, f"score.{sg}", Ln, rank=rank)).cuda()
              for sg, Ln in lens.items()}
        L.set_selection(nps, sc)
        L.X.copy_(dev(I.normal(seed, "x", h, N)))
        L.G.copy_(dev(I.normal(seed, "g", h, N)))
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            L.step(st)
            Z.ztp_sync(ctx, st)
            res.update(Y=host(L.Y), dX=host(L.dX), dqkv=host(L.dqkv), do=host(L.do), dw1=host(L.dw1[:, :u]),
                       dw2=host(L.dw2[:u]), nprune=np.array([nps[k] for k in ("qkv", "o", "fc1", "fc2")]))
            # the same step captured as a CUDA graph and replayed (peer kernels
            # carry their barrier epochs in device memory)
            L.Y.zero_()
            L.dX.zero_()
            g = L.capture(st)
            for _ in range(3):
                g.replay()
            Z.ztp_sync(ctx, st)
            res.update(Y_graph=host(L.Y), dX_graph=host(L.dX), dw1_graph=host(L.dw1[:, :u]))
    elif case == "kmig":
        # paper-literal K-dim migration of a column linear (NEXT-3): ranks in
        # PEER_MIGRATORS shed k contraction rows each, both policies
        from paper_2401_11469_b200.kmig import KMigColLinear
        K, n, N, seed = 256, 64, 136, 77
        migr = [int(v) for v in os.environ["PEER_MIGRATORS"].split(",")]
        k = int(os.environ["PEER_K"])
        mode = {"tree": Z.COLL_TREE, "p2p": Z.COLL_P2P}[os.environ["PEER_MODE"]]
        open_window(16 << 20)
        Lk = KMigColLinear(ctx, rank, world, K, n, N, migr, k, mode, alloc=sym_allocator(ctx, device))
        Lk.X.copy_(dev(I.normal(seed, "x", K, N)))
        Lk.W.copy_(dev(I.uniform_sym(seed, "w", K, world * n, 0.1, c0=rank * n, c1=(rank + 1) * n)))
        Lk.G.copy_(dev(I.normal(seed, "g", world * n, N, r0=rank * n, r1=(rank + 1) * n)))
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            Lk.step(st)
            Z.ztp_sync(ctx, st)
            res.update(Y=host(Lk.output()), dX=host(Lk.dX), dW=host(Lk.dW))
            # replayed as a CUDA graph
            Lk.dX.zero_()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                Lk.step(st)
            for _ in range(2):
                g.replay()
            Z.ztp_sync(ctx, st)
            res.update(Y_graph=host(Lk.output()), dX_graph=host(Lk.dX), dW_graph=host(Lk.dW))
    else:
        raise SystemExit(f"unknown case {case}")
    np.savez(os.path.join(out, f"{case}_{rank}.npz"), **res)
    dist.barrier()
    Z.ztp_ctx_destroy(ctx)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""The N > 1 host path on CPU with world_size 2 and 4 (gloo): every rank
gathers the statistics, runs ztp_plan / ztp_plan_counts (host library) and
gets the identical plan; the migration transfer lists built from it
(layer.migration_io / xfer_specs) are executed with point-to-point gloo copies
and move exactly the straggler's tail units into the helpers' appended slots
and the gradients back (A-26, A-27, A-28)."""
import math
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ztp_oracle as O


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stats(world, scenario):
    """Per-rank (T, M) of a statistics window with emulated slowdowns."""
    T, M = [], []
    for r in range(world):
        chi = 1.0
        if scenario == "single":
            chi = 3.0 if r == world - 1 else 1.0
        elif scenario == "multi":
            chi = {1: 8.0, 3: 6.0}.get(r, 1.0)
        m = 10.0 * chi
        T.append(m + 5.0)
        M.append(m)
    return T, M


def _worker(rank, world, port, scenario, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2401_11469_b200 as Z
        from paper_2401_11469_b200.layer import migration_io, xfer_specs
        h, f = 16, 64 * world
        u = f // world
        T_all, M_all = _stats(world, scenario)
        # every rank contributes only its own statistics (all-gather, Alg.2 l.2)
        mine = (T_all[rank], M_all[rank])
        got = [None] * world
        dist.all_gather_object(got, mine)
        T = [g[0] for g in got]
        M = [g[1] for g in got]
        lin = ((0.0, 1000.0), (0.0, 1.0))
        costs = Z.make_costs(0.0, lin, ((0.0, 1000.0), (0.0, 0.01)), ((0.0, 1000.0), (0.0, 0.01)))
        plan = Z.ztp_plan(T, M, float(u), costs, Z.plan_opts(enable_migration=1))
        key = (plan.z, plan.x, tuple(plan.role[:world]), tuple(plan.gamma[:world]), tuple(plan.beta[:world]),
               tuple(plan.phi[:world]), tuple(plan.gamma_r[:world]))
        keys = [None] * world
        dist.all_gather_object(keys, key)
        assert all(k == keys[0] for k in keys), "plans differ across ranks"
        mio = migration_io(plan, rank, world, u, h)
        cap = max([sum(hi - lo for (_, r, lo, hi, _) in
                       [(a, b, c, d, e) for (a, b, c, d, e) in mio.all_xfers if b == rr]) for rr in range(world)] + [1])
        # weights: own units hold rank-tagged values, appended slots NaN
        w1 = torch.full((h, u + cap), float("nan"))
        w2 = torch.full((u + cap, h), float("nan"))
        jj = torch.arange(u, dtype=torch.float64)
        w1[:, :u] = (rank * 1e4 + jj[None, :] + 0.5 * torch.arange(h)[:, None]).float()
        w2[:u] = (rank * 1e4 + jj[:, None] + 0.25 * torch.arange(h)[None, :]).float()
        tens = {"w1": w1, "w2": w2}

        def run(specs):
            ops, bufs = [], []
            for d in specs:
                t = tens[d["t"]]
                if d["src"] == rank and d["dst"] == rank:
                    t[d["dr0"]:d["dr0"] + d["nr"], d["dc0"]:d["dc0"] + d["nc"]] = \
                        t[d["r0"]:d["r0"] + d["nr"], d["c0"]:d["c0"] + d["nc"]].clone()
                elif d["src"] == rank:
                    buf = t[d["r0"]:d["r0"] + d["nr"], d["c0"]:d["c0"] + d["nc"]].contiguous()
                    ops.append(dist.P2POp(dist.isend, buf, d["dst"]))
                elif d["dst"] == rank:
                    buf = torch.empty(d["nr"], d["nc"])
                    bufs.append((d, buf))
                    ops.append(dist.P2POp(dist.irecv, buf, d["src"]))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for d, buf in bufs:
                tens[d["t"]][d["dr0"]:d["dr0"] + d["nr"], d["dc0"]:d["dc0"] + d["nc"]] = buf

        run(xfer_specs(mio, u, h, grads=False))
        # every received range holds exactly the owner's units
        off = 0
        for (src, lo, hi) in mio.inc:
            n = hi - lo
            exp1 = (src * 1e4 + torch.arange(lo, hi, dtype=torch.float64)[None, :]
                    + 0.5 * torch.arange(h)[:, None]).float()
            assert torch.equal(w1[:, u + off:u + off + n], exp1)
            exp2 = (src * 1e4 + torch.arange(lo, hi, dtype=torch.float64)[:, None]
                    + 0.25 * torch.arange(h)[None, :]).float()
            assert torch.equal(w2[u + off:u + off + n], exp2)
            off += n
        # gradients back: helper slots tagged with the helper rank
        dw1 = torch.zeros(h, u + cap)
        dw2 = torch.zeros(u + cap, h)
        dw1[:, u:] = 100.0 + rank
        dw2[u:] = 200.0 + rank
        tens.update(dw1=dw1, dw2=dw2)
        run(xfer_specs(mio, u, h, grads=True))
        for (dst, lo, hi) in mio.out:
            assert torch.all(dw1[:, lo:hi] == 100.0 + dst) and torch.all(dw2[lo:hi] == 200.0 + dst)
        # the migrated tail is [u - n_mig, u) and covered exactly once
        cov = [0] * u
        alls = [None] * world
        dist.all_gather_object(alls, [(s, lo, hi) for (s, lo, hi) in mio.inc])
        for lst in alls:
            for (s, lo, hi) in lst:
                if s == rank:
                    for j in range(lo, hi):
                        cov[j] += 1
        assert all(c == (1 if j >= u - mio.n_mig else 0) for j, c in enumerate(cov))
        # same plan as the oracle (bit-exact doubles)
        op = O.plan(T, M, float(u), O.Costs(0.0, lin, ((0.0, 1000.0), (0.0, 0.01)), ((0.0, 1000.0), (0.0, 0.01))),
                    O.PlanOpts(enable_migration=1))
        assert list(plan.role[:world]) == op.role and list(plan.gamma[:world]) == op.gamma
        q.put((rank, "ok", plan.z, plan.x, mio.n_mig, len(mio.inc)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"FAIL {type(e).__name__}: {e}", 0, 0, 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,scenario", [(2, "single"), (4, "single"), (4, "multi"), (2, "none")])
def test_multirank_plan_and_migration_gloo(world, scenario):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[1] == "ok", r
    if scenario == "single":
        s = [r for r in res if r[0] == world - 1][0]
        assert s[2] == 1 and s[4] > 0            # one straggler, migrating its tail
        assert sum(r[5] for r in res) == world - 1 or world == 2
    if scenario == "none":
        assert all(r[2] == 0 and r[4] == 0 for r in res)

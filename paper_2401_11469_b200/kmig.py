"""Paper-literal "sending-collecting" migration of a column-parallel linear
(Fig. 3): a migrating rank s sheds the
contraction rows J_s = [K - k, K) of its shard W_s^T [K, n] (the paper's
weight columns) to the normal ranks, which compute them for it.

  FWD   output of s: Y_s = W_s^T[K\\J]^T X^T[K\\J]  (s, a resized GEMM)
                         + sum_r W_s^T[J_r]^T X^T[J_r]  (helpers r, J_r a
                           renumbered range of J)
        the helpers' partials are COLLECTED to s (reduce / gather-sum).
  BWD   G_s (grad of s's output) is sent to the helpers; helper r adds
        W_s^T[J_r] G_s into rows J_r of its own dX partial before the
        all-reduce (the reduce merged into the all-reduce); helper r
        computes dW_s^T[J_r] = X^T[J_r] G_s^T and returns it to s.

Two communication policies (Table I):
  ZTP_COLL_TREE ("broadcast-reduce")  W_s^T[J] and G_s broadcast to every
        rank (each helper receives the whole migrated block and computes its
        share), partials collected by a reduce;
  ZTP_COLL_P2P  ("scatter-gather")    each helper receives only its rows
        J_r (point-to-point), G_s sent point-to-point, partials gathered
        point-to-point and summed by s.
Both compute the same result as the unsplit linear (migration is
loss-free).  Host orchestration only: every step runs in libztp
kernels and its collectives (the `ZtpLayer` migration of this build, A-26,
moves MLP hidden units instead; this module is the paper's per-linear form).
"""
from __future__ import annotations

from typing import List, Optional

import torch

import paper_2401_11469_b200 as Z


def helper_ranges(s: int, world: int, migrators: List[int], k: int):
    """Helpers of s = the NORMAL ranks (A-44), in r' = (r - s + e) mod e order
    (P:267); J = [0, k) split evenly, the remainder to the lowest r' (A-28).
    Returns [(r, a, b)] with local row ranges [a, b) of J."""
    helpers = sorted((r for r in range(world) if r not in migrators), key=lambda r: (r - s + world) % world)
    m, rem = divmod(k, len(helpers))
    out, a = [], 0
    for i, r in enumerate(helpers):
        c = m + (1 if i < rem else 0)
        out.append((r, a, a + c))
        a += c
    return out


class KMigColLinear:
    """One column-parallel linear of this rank with the paper-literal K-dim
    migration of the ranks in `migrators` (each sheds k rows of its K)."""

    def __init__(self, ctx, rank: int, world: int, K: int, n: int, N: int, migrators: List[int], k: int,
                 mode: int = Z.COLL_TREE, alloc=None, dtype=torch.bfloat16):
        if world > 1 and len(migrators) >= world:
            raise ValueError("every rank migrates: no helper")
        self.ctx, self.rank, self.world, self.K, self.n, self.N = ctx, rank, world, K, n, N
        self.migrators, self.k, self.mode, self.dtype = list(migrators), int(k), mode, dtype
        new = alloc or (lambda r, c, dt: torch.zeros(r, c, dtype=dt, device="cuda"))
        kk = max(self.k, 1)
        self.X = new(K, N, dtype)
        self.W = new(K, n, dtype)
        self.Y = new(n, N, dtype)
        self.G = new(n, N, dtype)
        self.dX = new(K, N, dtype)
        self.dW = new(K, n, dtype)
        self.T = new(kk, N, dtype)                 # a helper's migrated dX rows before the merge
        self.P, self.WJ, self.GS, self.DWJ = {}, {}, {}, {}
        for s in self.migrators:                  # per migrating rank (same on every rank: symmetric)
            self.P[s] = new(n, N, dtype)          # partial outputs of s's output, collected to s
            self.WJ[s] = new(kk, n, dtype)        # W_s^T[J] (broadcast) or rows J_r (scattered)
            self.GS[s] = new(n, N, dtype)         # G_s on the helpers
            self.DWJ[s] = new(kk, n, dtype)       # dW_s^T[J_r] computed by a helper
        self.iota = torch.arange(max(K, 1), dtype=torch.int32, device="cuda")
        self.empty = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._build()

    # ----------------------------------------------------------------- plan
    def _build(self):
        K, k, r = self.K, self.k, self.rank
        L = Z.linear_args
        self.ranges = {s: helper_ranges(s, self.world, self.migrators, k) for s in self.migrators}
        self.me_mig = r in self.migrators
        if self.me_mig:
            # own part: a resized GEMM over K \\ J (rows J pruned; dX / dW rows J Zero until the returns)
            self.sel_own = Z.sel(self.iota[:K - k], K - k, self.iota[K - k:], k, 90, 0)
            self.f_own = L(x_t=self.X, w_t=self.W, y_t=self.P[r], sel_=self.sel_own)
            self.b_own = L(x_t=self.X, w_t=self.W, g_t=self.G, dx_t=self.dX, dw_t=self.dW, sel_=self.sel_own,
                           skip_collective=1)
        else:
            self.f_own = L(x_t=self.X, w_t=self.W, y_t=self.Y)
            self.b_own = L(x_t=self.X, w_t=self.W, g_t=self.G, dx_t=self.dX, dw_t=self.dW, skip_collective=1)
        # helper work for each migrator: GEMMs over the local rows [a, b) of J
        self.help = []
        XJ = self.X[K - k:] if k else None
        for s in self.migrators:
            for (h, a, b) in self.ranges[s]:
                if h != r or b <= a:
                    continue
                kept = self.iota[a:b]
                pr = torch.cat([self.iota[:a], self.iota[b:k]]) if (a > 0 or b < k) else self.empty
                sl = Z.sel(kept, b - a, pr, k - (b - a), 91 + s, 0)
                self._keep = getattr(self, "_keep", []) + [pr]
                fa = L(x_t=XJ, w_t=self.WJ[s][:k], y_t=self.P[s], sel_=sl)
                ba = L(x_t=XJ, w_t=self.WJ[s][:k], g_t=self.GS[s], dx_t=self.T[:k], dw_t=self.DWJ[s][:k], sel_=sl)
                self.help.append((s, a, b, fa, ba))

    def _xfer(self, t, src, dst, r0, nr, dr0):
        return Z.xfer(t[0], t[1], r0=r0, c0=0, nr=nr, nc=t[0].shape[1], dr0=dr0, dc0=0, src_rank=src, dst_rank=dst)

    # ------------------------------------------------------------------ step
    def forward(self, stream=None):
        c, K, k = self.ctx, self.K, self.k
        Z.ztp_col_linear(c, Z.FWD, self.f_own, stream)
        for s in self.migrators:
            if self.mode == Z.COLL_TREE:
                # W_s^T[J] to every rank (s copies its rows J into its buffer first)
                Z.ztp_migrate(c, [self._xfer((self.W, self.WJ[s]), s, s, K - k, k, 0)], stream)
                Z.ztp_broadcast(c, s, self.WJ[s][:k], Z.COLL_TREE, stream)
            else:
                xs = [self._xfer((self.W, self.WJ[s]), s, h, K - k + a, b - a, a) for (h, a, b) in self.ranges[s]]
                Z.ztp_migrate(c, xs, stream)
        for (s, a, b, fa, ba) in self.help:
            Z.ztp_gemm(c, Z.KIND_FWD, fa, stream)
        for s in self.migrators:
            Z.ztp_reduce(c, s, self.P[s], self.mode, stream)     # s's output = its own part + the helpers'

    def output(self):
        return self.P[self.rank] if self.me_mig else self.Y

    def backward(self, stream=None):
        c, K, k = self.ctx, self.K, self.k
        for s in self.migrators:
            # G_s to the helpers (broadcast, or point-to-point copies of the whole G_s)
            Z.ztp_migrate(c, [self._xfer((self.G, self.GS[s]), s, s, 0, self.n, 0)], stream)
            Z.ztp_broadcast(c, s, self.GS[s], self.mode, stream)
        Z.ztp_col_linear(c, Z.BWD, self.b_own, stream)          # own dX partial + own dW (skip the all-reduce)
        for (s, a, b, fa, ba) in self.help:
            Z.ztp_gemm(c, Z.KIND_DX, ba, stream)                 # rows J_r of W_s^T[J] G_s (others Zero)
            Z.ztp_gemm(c, Z.KIND_DW, ba, stream)                 # dW_s^T[J_r] rows
            Z.ztp_accumulate(c, self.dX[K - k + a:K - k + b], self.T[a:b], stream)   # merged into the partial
        Z.ztp_allreduce(c, self.dX, stream)
        xs = []
        for s in self.migrators:                                  # dW_s^T[J_r] back to s's rows J
            xs += [self._xfer((self.DWJ[s], self.dW), h, s, a, b - a, K - k + a) for (h, a, b) in self.ranges[s]
                   if b > a]
        if xs:
            Z.ztp_migrate(c, xs, stream)
        Z.ztp_join(c, stream)                                     # the concurrent own dW ends the step

    def step(self, stream=None):
        self.forward(stream)
        self.backward(stream)

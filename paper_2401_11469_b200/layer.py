"""One transformer layer of 1D tensor parallelism on this rank, driven through
the C ABI (SURVEY §8(a) "Layer definition used for measurement"):

  attention-projection block: QKV (col) -> stand-in core ctx = Q+K+V (A-31)
                              -> O (row) -> all-reduce
  MLP block:                  FC1 (col) -> GeLU -> FC2 (row) -> all-reduce

Every tensor is feature-major ([features, tokens]) and every weight is stored
W^T [K, n].  This module only allocates device buffers
(torch, as plumbing), builds the ztp_linear_args structs once, and issues the
call sequence of a step; all arithmetic runs in libztp.so kernels and NCCL.

Producer-side compaction: the core writes ctx only for O's kept
rows S_o (compact), FC1's epilogue writes pre/H only for FC2's kept rows S_w
(compact, through FC2's inverse map), and the col layers' inputs X / Y1 are
compacted once in FWD (xs buffers) and reused in BWD.  So every GEMM mainloop
streams dense TMA boxes.

Migration (SEMI, A-26): a helper holds W1^T / W2^T with spare capacity; the
straggler's hidden units J are pulled into the appended columns / rows
(ztp_migrate) and simply extend the helper's FC1 output and FC2 contraction
(kept list S_w + appended indices) -- the local reduce is the same TMEM
accumulator, merged into the existing all-reduces.  dW slices of J
are pushed back to the owner after BWD.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import os
from typing import Dict, List, Optional

import torch

import paper_2401_11469_b200 as Z

SEGS = ("qkv", "o", "fc1", "fc2")


def _buf(r, c, dtype=torch.bfloat16, fill=0.0):
    """Row pitch padded to 16 bytes (TMA stride rule)."""
    ld = (c + 7) // 8 * 8
    t = torch.full((max(r, 1), ld), fill, dtype=dtype, device="cuda")
    return t[:, :c]


def _on(stream):
    """torch work on the library's stream (the fused attention core)."""
    import contextlib
    return torch.cuda.stream(stream) if isinstance(stream, torch.cuda.Stream) else contextlib.nullcontext()


def sym_allocator(ctx, device: int = 0):
    """Allocator of window tensors (ztp_sym_alloc; zero-filled at window
    creation) for ZtpLayer(alloc=...) under the peer transport."""
    return lambda r, c, dtype: Z.ztp_sym_alloc(ctx, r, c, dtype, device)


@dataclass
class AttnSpec:
    """The real attention core (NEXT-4; replaces A-31's stand-in): heads of
    head_dim features, tokens t = batch * seq + s, causal or not.  The fused
    attention itself is cuDNN's (through torch SDPA: a library kernel like
    cuBLAS, the core being outside the method, A-31); the layout changes
    around it are libztp's ztp_transpose."""
    head_dim: int
    seq: int
    causal: bool = True


@dataclass
class MigrationIO:
    """This rank's migration ranges from ztp_plan_counts (FC1/FC2 units)."""
    n_mig: int = 0                                     # my units shed (tail)
    out: List[tuple] = field(default_factory=list)     # (dst, lo, hi)
    inc: List[tuple] = field(default_factory=list)     # (src, lo, hi)
    all_xfers: List[tuple] = field(default_factory=list)  # (src, dst, lo, hi, dst_off) for every pair


def migration_io(plan, rank: int, world: int, u: int, h: int, unit: int = 1) -> MigrationIO:
    """This rank's migration I/O from a plan, via ztp_plan_counts (host only).
    all_xfers lists every (src, dst, lo, hi, dst_off) pair of the layer so all
    ranks issue the same ztp_migrate list; dst_off is the offset of the range
    inside the helper's appended slots [u, u + cap)."""
    counts = [Z.ztp_plan_counts(plan, r, u, u, unit, True) for r in range(world)]
    me = counts[rank]
    mio = MigrationIO(n_mig=me.n_mig,
                      out=[(me.out_dst[i], me.out_lo[i], me.out_hi[i]) for i in range(me.n_out)],
                      inc=[(me.in_src[i], me.in_lo[i], me.in_hi[i]) for i in range(me.n_in)])
    for r in range(world):
        off = 0
        c = counts[r]
        for i in range(c.n_in):
            lo, hi = c.in_lo[i], c.in_hi[i]
            mio.all_xfers.append((c.in_src[i], r, lo, hi, off))
            off += hi - lo
    return mio


def layer_prune_counts(plan, rank: int, h: int, a: int, u: int) -> Dict[str, int]:
    """Prune counts of the four linears of `rank` from a plan: the library's
    ztp_layer_prune_counts (MLP by gamma_r, attention by the A-37 rule)."""
    return Z.ztp_layer_prune_counts(plan, rank, h, a, u)


def xfer_specs(mio: MigrationIO, u: int, h: int, grads: bool) -> List[dict]:
    """Peer copies of one layer's migration (pure host logic).  Weights: the
    owner's units [lo, hi) -> the helper's appended slots [u+off, ...) of W1^T
    (columns) and W2^T (rows).  Gradients: the reverse, into dW1^T / dW2^T."""
    out = []
    for (src, dst, lo, hi, off) in mio.all_xfers:
        n = hi - lo
        if not grads:
            out.append(dict(t="w1", src=src, dst=dst, r0=0, c0=lo, nr=h, nc=n, dr0=0, dc0=u + off))
            out.append(dict(t="w2", src=src, dst=dst, r0=lo, c0=0, nr=n, nc=h, dr0=u + off, dc0=0))
        else:
            out.append(dict(t="dw1", src=dst, dst=src, r0=0, c0=u + off, nr=h, nc=n, dr0=0, dc0=lo))
            out.append(dict(t="dw2", src=dst, dst=src, r0=u + off, c0=0, nr=n, nc=h, dr0=lo, dc0=0))
    return out


class ZtpLayer:
    def __init__(self, ctx, h: int, f: int, N: int, rank: int, world: int, shards: Optional[Dict[str, torch.Tensor]],
                 mig_cap: int = 0, dtype=torch.bfloat16, layer_id: int = 0, alloc=None, plain: bool = False,
                 attn: Optional[AttnSpec] = None):
        """alloc(rows, cols, dtype) -> zero-filled tensor: where the layer's
        buffers live (default torch; `sym_allocator(ctx)` for the peer
        transport, whose all-reduce and migration operands must be window
        tensors at the same offsets on every rank).
        plain (always so for dtype float32, the verification mode A-30): no
        producer-side compaction and no output pruning -- every activation
        is kept at full size, the GEMMs read kept rows through the lineage
        and the epilogues write / zero-impute rows at their positions."""
        self.ctx, self.h, self.f, self.N = ctx, h, f, N
        self.rank, self.world = rank, world
        # the O projection's dW after the core (beside the QKV backward) instead of beside its own dX
        # (dw_side): O dX then runs alone on every SM; profiles/r02_late_o_dw_ab.txt
        self.late_o_dw = os.environ.get("ZTP_LATE_O_DW", "0") != "0"   # measured slower at c2: opt-in
        self.a = h // world                  # attention features per rank
        self.u = f // world                  # MLP hidden units per rank
        self.cap = mig_cap
        self.dtype = dtype
        self.layer_id = layer_id
        self.alloc = alloc
        self.plain = plain or dtype == torch.float32
        self.attn = attn
        if attn is not None:
            if dtype != torch.bfloat16 or (h // world) % attn.head_dim or N % attn.seq:
                raise ValueError("attention core: bf16, whole heads per rank, whole sequences")
            # token-major copies for the fused attention ([batch, seq, heads, head_dim])
            self.QKVt = torch.zeros(N, 3 * (h // world), dtype=dtype, device="cuda")
            self.dOt = torch.zeros(N, h // world, dtype=dtype, device="cuda")
        a, u, cap = self.a, self.u, mig_cap
        for name, r, c in self.buffer_specs(h, f, N, world, mig_cap):
            setattr(self, name, self._new(r, c))
        if shards is not None:
            self.qkv_t.copy_(shards["qkv"])
            self.o_t.copy_(shards["o"])
            self.w1_t[:, :u].copy_(shards["w1"])
            self.w2_t[:u].copy_(shards["w2"])
        # selection buffers (lineage)
        self.K = {"qkv": h, "o": a, "fc1": h, "fc2": u + cap}
        total = sum(self.K.values()) + 3 * a        # + the derived V-output segment (A-36)
        self.kept = torch.zeros(total, dtype=torch.int32, device="cuda")
        self.pruned = torch.zeros(total, dtype=torch.int32, device="cuda")
        self.pos = torch.zeros(total + cap, dtype=torch.int32, device="cuda")
        self.mig = MigrationIO()
        self.n_fc = u                            # FC1 output units computed / FC2 K
        self.set_selection({s: 0 for s in SEGS}, None)

    @staticmethod
    def buffer_specs(h: int, f: int, N: int, world: int, cap: int):
        """(attribute, rows, cols) of every device buffer, in allocation order
        (identical on every rank, so window offsets are symmetric)."""
        a, u = h // world, f // world
        return [
            # weights (W^T), MLP ones with migration capacity
            ("qkv_t", h, 3 * a), ("o_t", a, h), ("w1_t", h, u + cap), ("w2_t", u + cap, h),
            # activations: X, compact X rows S_qkv, QKV, compact ctx rows S_o, Y1,
            # compact Y1 rows S_fc1, compact GeLU'(pre) / H rows S_fc2, Y
            ("X", h, N), ("Xc", h, N), ("QKV", 3 * a, N), ("ctxC", a, N), ("Y1", h, N), ("Y1c", h, N),
            ("PreC", u + cap, N), ("HC", u + cap, N), ("Y", h, N),
            # gradients (G1 = dH * GeLU'(pre), compact rows S_fc2)
            ("G", h, N), ("G1", u + cap, N), ("dY1", h, N), ("dctx", a, N), ("gQKV", 3 * a, N), ("dX", h, N),
            ("dqkv", h, 3 * a), ("do", a, h), ("dw1", h, u + cap), ("dw2", u + cap, h),
            # compact weights
            ("Wqkv_c", h, 3 * a), ("Wo_c", a, h), ("W1_c", h, u + cap), ("W2_c", u + cap, h),
        ]

    @staticmethod
    def window_bytes(h: int, f: int, N: int, world: int, cap: int = 0, es: int = 2) -> int:
        """Symmetric-window bytes the layer's buffers take (ztp_sym_alloc
        rounds every allocation to 256 bytes)."""
        tot = 0
        for _, r, c in ZtpLayer.buffer_specs(h, f, N, world, cap):
            ld = (c * es + 15) // 16 * 16 // es
            tot += (max(r, 1) * ld * es + 255) // 256 * 256
        return tot

    def _new(self, r, c):
        if self.alloc is not None:
            return self.alloc(r, c, self.dtype)
        return _buf(r, c, self.dtype)

    # ------------------------------------------------------------------ plan
    def set_migration(self, mio: MigrationIO):
        """Apply this rank's migration ranges (from ztp_plan_counts)."""
        self.mig = mio
        n_in = sum(hi - lo for (_, lo, hi) in mio.inc)
        if n_in > self.cap:
            raise ValueError(f"migration needs {n_in} units of capacity, have {self.cap}")
        self.n_fc = self.u - mio.n_mig + n_in

    def set_selection(self, n_prune: Dict[str, int], scores: Optional[Dict[str, torch.Tensor]],
                      stream=None):
        """Run ztp_select for the four segments (one launch) and rebuild the
        lineage entries and argument structs.  n_prune['fc2'] counts only my own
        (non-migrated) units; received units are appended (never pruned)."""
        own_fc2 = self.u - self.mig.n_mig
        n_in = self.n_fc - own_fc2
        self.seg_len = {"qkv": self.h, "o": self.a, "fc1": self.h, "fc2": own_fc2}
        self.append = {"qkv": 0, "o": 0, "fc1": 0, "fc2": n_in}
        self.n_prune = dict(n_prune)
        # A-36: the V rows of the QKV output feed only ctx features S_o (the
        # O projection's kept set), so QKV computes V for S_o only.  The V
        # selection is a derived segment over the 3a QKV outputs -- Q and K
        # scored +inf (never pruned), V scored like O's inputs -- selected in
        # the same launch, so it is exactly O's (S_o, P_o) shifted by 2a.
        self.v_prune = (self.n_prune["o"] > 0 and os.environ.get("ZTP_V_PRUNE", "1") != "0" and not self.plain
                        and self.attn is None)
        segs = SEGS + (("vo",) if self.v_prune else ())
        if self.v_prune:
            self.seg_len["vo"], self.append["vo"], self.n_prune["vo"] = 3 * self.a, 0, self.n_prune["o"]
        lens = [self.seg_len[s] for s in segs]
        nps = [self.n_prune[s] for s in segs]
        apps = [self.append[s] for s in segs]
        if scores is None:
            base = [torch.zeros(self.seg_len[s], dtype=torch.float32, device="cuda") for s in SEGS]
        else:
            base = [scores[s][: self.seg_len[s]].float() for s in SEGS]
        if self.v_prune:
            inf = torch.full((2 * self.a,), float("inf"), dtype=torch.float32, device="cuda")
            base = base + [inf, base[1]]
        sc = torch.cat(base)
        self._scores = sc
        self._sel_args = (lens, nps, apps)
        self.run_select(stream)
        # slices of the lineage buffers
        ko = po = qo = 0
        self.S, self.P, self.POS, self.nk = {}, {}, {}, {}
        for s in segs:
            nk = self.seg_len[s] - self.n_prune[s] + self.append[s]
            self.S[s] = self.kept[ko:ko + nk]
            self.P[s] = self.pruned[po:po + max(self.n_prune[s], 0)]
            self.POS[s] = self.pos[qo:qo + self.seg_len[s] + self.append[s]]
            self.nk[s] = nk
            ko += nk
            po += self.n_prune[s]
            qo += self.seg_len[s] + self.append[s]
        self._build_args()

    def weight_rows(self) -> Dict[str, torch.Tensor]:
        """W^T of each segment restricted to the rows the segment selects over
        (own units only for FC2)."""
        own = self.u - self.mig.n_mig
        return {"qkv": self.qkv_t, "o": self.o_t, "fc1": self.w1_t[:, :self.u], "fc2": self.w2_t[:own]}

    def priority_epoch(self, w_prev: Dict[str, torch.Tensor], gamma_t: float, theta: float,
                       alpha: float = 0.8, stream=None) -> Dict[str, int]:
        """NEXT-1, once per epoch (Alg.1 l.3-14): per segment, the column
        variation of W^T against the previous epoch's weights (pruned rows keep
        their score), the PriDiff ratio max(1 - L_uni/L, alpha gamma_t)
        (l.9-11) and the new selection on the maintained scores (l.12-14).
        Returns the per-segment prune counts."""
        cur = self.weight_rows()
        lens = {s: self.seg_len[s] for s in SEGS}
        offs, o = {}, 0
        for s in SEGS:
            offs[s] = o
            o += lens[s]
        cnt = torch.zeros(len(SEGS), dtype=torch.int32, device="cuda")
        first = not getattr(self, "_prio_init", False)
        for i, s in enumerate(SEGS):
            delta = self._scores[offs[s]:offs[s] + lens[s]]
            pos = None if first else self.POS[s][:lens[s]]
            Z.ztp_priority_update(self.ctx, cur[s], w_prev[s], delta, pos_prev=pos, count_above=cnt[i:i + 1],
                                  theta=theta, stream=stream)
        self._prio_init = True
        l_uni = cnt.cpu().tolist()                 # epoch boundary: one host sync
        n_prune = {}
        for i, s in enumerate(SEGS):
            n_prune[s] = Z.ztp_pridiff_counts(lens[s], l_uni[i], gamma_t, alpha, 0.9)   # l.10-11, A-3, A-4
        scores = {s: self._scores[offs[s]:offs[s] + lens[s]].clone() for s in SEGS}
        self.set_selection(n_prune, scores, stream)
        return n_prune

    def run_select(self, stream=None):
        lens, nps, apps = self._sel_args
        Z.ztp_select(self.ctx, lens, nps, self._scores, self.kept, self.pruned, apps, self.pos, stream)

    def _sel(self, s, mid):
        if self.n_prune[s] == 0 and (self.append[s] == 0 or s == "fc2"):
            # dense: no lineage entry, operands used in place.  A helper's
            # received MLP units sit right after its own ones (W1^T columns /
            # W2^T rows u .. u + n_in), so an unpruned FC2 with appended units
            # is the dense prefix of length n_fc -- no compaction copies
            return None
        p = self.P[s] if self.n_prune[s] > 0 else self.kept
        return Z.sel(self.S[s], self.nk[s], p, self.n_prune[s], self.layer_id, mid)

    def _build_args_plain(self):
        """Argument structs of the plain arrangement (see __init__)."""
        h, a, N, nfc = self.h, self.a, self.N, self.n_fc
        L = Z.linear_args
        self.vsel, self.y1_direct, self._prep = None, False, []
        sl = self.sels
        self.f_qkv = L(x_t=self.X, w_t=self.qkv_t, y_t=self.QKV, sel_=sl["qkv"], n_out=3 * a)
        self.f_o = L(x_t=self.ctxC, w_t=self.o_t, y_t=self.Y1, sel_=sl["o"])
        self.f_fc1 = L(x_t=self.Y1, w_t=self.w1_t, y_t=self.HC[:nfc], pre_t=self.PreC[:nfc], sel_=sl["fc1"],
                       n_out=nfc, act=Z.ACT_GELU_D)
        self.f_fc2 = L(x_t=self.HC[:nfc], w_t=self.w2_t[:nfc], y_t=self.Y, sel_=sl["fc2"])
        self.b_fc2 = L(x_t=self.HC[:nfc], w_t=self.w2_t[:nfc], g_t=self.G, dx_t=self.G1[:nfc], dw_t=self.dw2[:nfc],
                       pre_in_t=self.PreC[:nfc], sel_=sl["fc2"], act_in=Z.ACT_GELU_D)
        self.b_fc1 = L(x_t=self.Y1, w_t=self.w1_t, g_t=self.G1[:nfc], dx_t=self.dY1, dw_t=self.dw1, sel_=sl["fc1"],
                       n_out=nfc)
        self.b_o = L(x_t=self.ctxC, w_t=self.o_t, g_t=self.dY1, dx_t=self.dctx, dw_t=self.do, sel_=sl["o"])
        self.b_o_dx = self.b_o_dw = None
        self.b_qkv = L(x_t=self.X, w_t=self.qkv_t, g_t=self.gQKV, dx_t=self.dX, dw_t=self.dqkv, sel_=sl["qkv"],
                       n_out=3 * a)

    def _build_args(self):
        h, a, N, nfc = self.h, self.a, self.N, self.n_fc
        self.sels = {s: self._sel(s, i) for i, s in enumerate(SEGS)}
        if self.plain:
            return self._build_args_plain()
        vsel = self._sel("vo", 4) if self.v_prune else None
        self.vsel = vsel
        L = Z.linear_args
        nk = self.nk
        ngq = 2 * a + nk["o"] if vsel is not None else 3 * a      # QKV output rows computed
        # forward
        vkw = {"out_sel": vsel, "y_pos": self.POS["vo"]} if vsel is not None else {}
        self.f_qkv = L(x_t=self.X, w_t=self.qkv_t, y_t=self.QKV, xs_t=self.Xc, ws_t=self.Wqkv_c,
                       sel_=self.sels["qkv"], n_out=3 * a, **vkw)
        # TP = 1 (no all-reduce of Y1): the O projection's epilogue writes Y1
        # directly in FC1's kept order (rows S_fc1, through its inverse map),
        # so no full Y1 and no compaction copy exist.  TP > 1 all-reduces the
        # full Y1 first (ranks keep different S_fc1), then FC1 compacts.
        self.y1_direct = (self.world == 1 and self.sels["fc1"] is not None
                          and os.environ.get("ZTP_Y1_DIRECT", "1") != "0")   # A/B knob
        if self.y1_direct:
            y1, y1_kw = self.Y1c[:nk["fc1"]], {"x_compact": True}
            self.f_o = L(x_t=self.ctxC[:nk["o"]], w_t=self.o_t, y_t=self.Y1c, ws_t=self.Wo_c, sel_=self.sels["o"],
                         x_compact=True, y_pos=self.POS["fc1"])
        else:
            y1, y1_kw = self.Y1, {"xs_t": self.Y1c}
            self.f_o = L(x_t=self.ctxC[:nk["o"]], w_t=self.o_t, y_t=self.Y1, ws_t=self.Wo_c, sel_=self.sels["o"],
                         x_compact=True)
        # output pruning: FC1 computes only the hidden units FC2 keeps (S_fc2)
        # and its backward reads the compact G1 FC2's dX writes (rows P_fc2
        # are Zero) -- same results as the full FC1, half the work at
        # gamma = 0.5.  DESIGN.md "Output pruning".
        osel = self.sels["fc2"]
        ng = nk["fc2"] if osel is not None else nfc
        self.f_fc1 = L(x_t=y1, w_t=self.w1_t, y_t=self.HC, pre_t=self.PreC, ws_t=self.W1_c,
                       sel_=self.sels["fc1"], n_out=nfc, act=Z.ACT_GELU_D, y_pos=self.POS["fc2"] if osel is not None else None,
                       out_sel=osel,
                       **y1_kw)
        self.f_fc2 = L(x_t=self.HC[:nk["fc2"]], w_t=self.w2_t[:nfc], y_t=self.Y, ws_t=self.W2_c,
                       sel_=self.sels["fc2"], x_compact=True)
        # batched compaction (ztp_prepare): X + Wqkv, Wo, W1 (2D), W2
        self._prep = []
        for args, what in ((self.f_qkv, 3), (self.f_o, 2), (self.f_fc1, 2), (self.f_fc2, 2)):
            if args.sel or args.out_sel:
                args.prepared = what
                self._prep.append((args, what))
        # backward
        self.b_fc2 = L(x_t=self.HC[:nk["fc2"]], w_t=self.w2_t[:nfc], g_t=self.G, dx_t=self.G1[:ng],
                       dw_t=self.dw2[:nfc], pre_in_t=self.PreC[:nk["fc2"]], ws_t=self.W2_c,
                       sel_=self.sels["fc2"], act_in=Z.ACT_GELU_D, x_compact=True, dx_compact=osel is not None)
        self.b_fc1 = L(x_t=y1, w_t=self.w1_t, g_t=self.G1[:ng], dx_t=self.dY1, dw_t=self.dw1,
                       ws_t=self.W1_c, sel_=self.sels["fc1"], n_out=nfc, y_pos=self.POS["fc2"] if osel is not None else None,
                       out_sel=osel,
                       **y1_kw)
        self.b_o = L(x_t=self.ctxC[:nk["o"]], w_t=self.o_t, g_t=self.dY1, dx_t=self.dctx, dw_t=self.do,
                     ws_t=self.Wo_c, sel_=self.sels["o"], x_compact=True)
        # late O dW: dX alone on every SM, the core, then dW on the side stream beside the QKV backward
        self.b_o_dx = L(x_t=self.ctxC[:nk["o"]], w_t=self.o_t, g_t=self.dY1, dx_t=self.dctx,
                        ws_t=self.Wo_c, sel_=self.sels["o"], x_compact=True)
        self.b_o_dw = L(x_t=self.ctxC[:nk["o"]], w_t=self.o_t, g_t=self.dY1, dw_t=self.do,
                        ws_t=self.Wo_c, sel_=self.sels["o"], x_compact=True, dw_side=True)
        self.b_qkv = L(x_t=self.X, w_t=self.qkv_t, g_t=self.gQKV[:ngq], dx_t=self.dX, dw_t=self.dqkv, xs_t=self.Xc,
                       ws_t=self.Wqkv_c, sel_=self.sels["qkv"], n_out=3 * a, **vkw)

    # --------------------------------------------------------------- migration
    def _xfers(self, grads: bool):
        tens = {"w1": self.w1_t, "w2": self.w2_t, "dw1": self.dw1, "dw2": self.dw2}
        xs = []
        for d in xfer_specs(self.mig, self.u, self.h, grads):
            t = tens[d["t"]]
            # every rank passes its own tensor as both ends: the source rank's
            # is read (NCCL: packed and sent), the destination rank's is written,
            # and under the peer transport the destination's own counterpart of
            # the source locates the slice in the source rank's window
            xs.append(Z.xfer(t, t,
                             r0=d["r0"], c0=d["c0"], nr=d["nr"], nc=d["nc"], dr0=d["dr0"], dc0=d["dc0"],
                             src_rank=d["src"], dst_rank=d["dst"]))
        return xs

    def migrate_weights(self, stream=None):
        if self.mig.all_xfers:
            Z.ztp_migrate(self.ctx, self._xfers(False), stream)

    def return_grads(self, stream=None):
        if self.mig.all_xfers:
            Z.ztp_migrate(self.ctx, self._xfers(True), stream)

    # -------------------------------------------------------------------- step
    def prepare(self, stream=None):
        """All compact operand copies that depend only on the step's inputs,
        weights and selection (X rows S_qkv, and the weight blocks of the four
        linears) in one launch; the FWD calls then skip their own copies."""
        if self._prep:
            Z.ztp_prepare(self.ctx, self._prep, stream)

    def fwd_attn(self, stream=None):
        c = self.ctx
        self.prepare(stream)
        Z.ztp_col_linear(c, Z.FWD, self.f_qkv, stream)
        if self.attn is not None:
            self._attn_fwd(stream)
        elif self.plain:   # ctx at full size, O reads its kept rows through the lineage
            Z.ztp_core(c, Z.FWD, self.QKV, self.ctxC, self.a, self.a, None, 0, stream)
        else:              # ctx written compact in O's kept order
            Z.ztp_core(c, Z.FWD, self.QKV, self.ctxC, self.a, self.a, self.S["o"], self.nk["o"], stream,
                       v_compact=self.vsel is not None)
        Z.ztp_row_linear(c, Z.FWD, self.f_o, stream)          # + all-reduce of Y1

    def fwd_mlp(self, stream=None):
        c = self.ctx
        Z.ztp_col_linear(c, Z.FWD, self.f_fc1, stream)        # GeLU epilogue, compact rows S_fc2
        Z.ztp_row_linear(c, Z.FWD, self.f_fc2, stream)        # + all-reduce of Y

    def bwd_mlp(self, stream=None):
        c = self.ctx
        Z.ztp_row_linear(c, Z.BWD, self.b_fc2, stream)        # dH -> G1 = dH * GeLU'(pre), dW2
        Z.ztp_col_linear(c, Z.BWD, self.b_fc1, stream)        # dY1 (+ all-reduce), dW1

    def _heads(self, t):
        """[N, k * a] token-major -> k views [batch, heads, seq, head_dim]."""
        sp = self.attn
        B, S, H, D = self.N // sp.seq, sp.seq, self.a // sp.head_dim, sp.head_dim
        k = t.shape[1] // self.a
        v = t.view(B, S, k, H, D)
        return [v[:, :, i].transpose(1, 2) for i in range(k)]

    def _attn_fwd(self, stream=None):
        """Real core FWD: QKV^T -> token-major (ztp_transpose), fused causal /
        bidirectional attention (cuDNN), output -> ctx^T in O's kept order S_o."""
        import torch.nn.functional as F
        from torch.nn.attention import SDPBackend, sdpa_kernel
        c, N, a = self.ctx, self.N, self.a
        Z.ztp_transpose(c, self.QKV, self.QKVt, None, N, stream)
        self._qkv_leaf = self.QKVt.detach().requires_grad_(True)
        q, k, v = self._heads(self._qkv_leaf)
        with _on(stream), torch.enable_grad(), sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            self._o = F.scaled_dot_product_attention(q, k, v, is_causal=self.attn.causal)
            ot = self._o.transpose(1, 2).reshape(N, a)
        Z.ztp_transpose(c, ot, self.ctxC, self.S["o"], self.nk["o"], stream)

    def _attn_bwd(self, stream=None):
        """Real core BWD: dctx^T -> token-major dO, the fused attention
        backward (cuDNN) -> dQKV token-major -> gQKV^T (ztp_transpose)."""
        c, N = self.ctx, self.N
        Z.ztp_transpose(c, self.dctx, self.dOt, None, N, stream)
        do = self._heads(self.dOt)[0]
        with _on(stream):
            (dqkv,) = torch.autograd.grad(self._o, self._qkv_leaf, do)
        Z.ztp_transpose(c, dqkv, self.gQKV, None, 3 * self.a, stream)
        self._o = self._qkv_leaf = None

    def bwd_attn(self, stream=None):
        c = self.ctx
        late = self.late_o_dw and self.b_o_dw is not None
        Z.ztp_row_linear(c, Z.BWD, self.b_o_dx if late else self.b_o, stream)   # dctx (+ dWo beside it)
        if self.attn is not None:
            self._attn_bwd(stream)
        elif self.vsel is not None:
            Z.ztp_core(c, Z.BWD, self.gQKV, self.dctx, self.a, self.a, self.S["o"], self.nk["o"], stream,
                       v_compact=True)
        else:
            Z.ztp_core(c, Z.BWD, self.gQKV, self.dctx, self.a, self.a, None, 0, stream)
        if late:
            Z.ztp_row_linear(c, Z.BWD, self.b_o_dw, stream)   # dWo on the side stream
        Z.ztp_col_linear(c, Z.BWD, self.b_qkv, stream)        # dX (+ all-reduce), dWqkv
        Z.ztp_join(c, stream)                                  # concurrent dW work (ZTP_CONC) ends the step

    def forward(self, stream=None):
        self.fwd_attn(stream)
        self.fwd_mlp(stream)

    def backward(self, stream=None):
        self.bwd_mlp(stream)
        self.bwd_attn(stream)

    def step(self, stream=None, select: bool = True):
        """One pass of the hot path: (select) + migrate weights + FWD + BWD +
        return migrated weight gradients."""
        if select:
            self.run_select(stream)
        self.migrate_weights(stream)
        self.forward(stream)
        self.backward(stream)
        self.return_grads(stream)

    def capture(self, stream, select: bool = True, pre=None, post=None):
        """Record one step (optionally wrapped by `pre`/`post` callables, e.g.
        host<->device copies) into a CUDA graph on `stream` (a non-default
        torch stream).  The library launches nothing that allocates or syncs in
        steady state, so the whole step -- select, GEMMs, epilogues, NCCL --
        is captured; replay() re-issues it with one launch."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            if pre is not None:
                pre()
            self.step(stream, select=select)
            if post is not None:
                post()
        self._graph = g
        return g

    def replay(self):
        self._graph.replay()

    # ------------------------------------------------------------ accounting
    def method_flops(self) -> float:
        """FLOPs of the resized layer by the method's count: 6 N n K' per
        linear (fwd + dX + dW), SURVEY §8(d)."""
        N, a, h = self.N, self.a, self.h
        nk = self.nk
        return 6.0 * N * (3 * a * nk["qkv"] + h * nk["o"] + self.n_fc * nk["fc1"] + h * nk["fc2"])

    def executed_flops(self) -> float:
        """FLOPs the GEMMs of one step execute: as method_flops, except that
        FC1 computes only the units FC2 keeps (A-35) and QKV computes V only
        for O's kept features (A-36) -- same results, less work."""
        N, a, h = self.N, self.a, self.h
        nk = self.nk
        n_qkv = 2 * a + nk["o"] if self.vsel is not None else 3 * a
        n_fc1 = nk["fc2"] if self.sels["fc2"] is not None else self.n_fc
        return 6.0 * N * (n_qkv * nk["qkv"] + h * nk["o"] + n_fc1 * nk["fc1"] + h * nk["fc2"])


class ZtpStack:
    """Several layers of one rank run as one step: per layer the weight
    migration pulls (SEMI plans), then the forward of every layer, the
    backward in reverse order, and the migrated dW slices returned.  The
    selection runs once per plan (set_selection; the priority list is
    epoch-granular), not inside the step."""

    def __init__(self, layers: List[ZtpLayer]):
        self.layers = layers

    def step(self, stream=None, select: bool = False):
        for L in self.layers:
            if select:
                L.run_select(stream)
            L.migrate_weights(stream)
        for L in self.layers:
            L.forward(stream)
        for L in reversed(self.layers):
            L.backward(stream)
        for L in self.layers:
            L.return_grads(stream)

    def capture(self, stream, select: bool = False, pre=None, post=None):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            if pre is not None:
                pre()
            self.step(stream, select=select)
            if post is not None:
                post()
        return g

    def method_flops(self) -> float:
        return sum(L.method_flops() for L in self.layers)

    def executed_flops(self) -> float:
        return sum(L.executed_flops() for L in self.layers)

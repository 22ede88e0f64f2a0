"""Workload shapes of BASELINE.json `configs`.  Shapes and the
emulated per-rank slowdowns only -- no arithmetic of the method."""
from __future__ import annotations

from dataclasses import dataclass, field

from .inputs import BASE_SEED


@dataclass(frozen=True)
class LayerConfig:
    name: str
    index: int          # config index (seed = BASE_SEED + index)
    h: int              # hidden size
    f: int              # FFN inner size
    heads: int
    N: int              # tokens = batch * seq
    mlp_only: bool = False
    layers: int = 1
    note: str = ""
    seq: int = 0        # tokens per sequence (N = batch * seq), for the real attention core
    causal: bool = True # decoder (GPT / Llama) vs encoder (ViT) attention

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index

    @property
    def head_dim(self) -> int:
        return self.h // self.heads


CONFIGS = {
    # c1: single FFN block h=64 f=256 seq16 x batch2, TP=2, rank1 2x, gamma 0.25
    "c1": LayerConfig("c1", 0, h=64, f=256, heads=1, N=32, mlp_only=True,
                      note="single FFN block h=64 ffn=256 seq=16 batch=2", seq=16),
    # c2: GPT-2 medium layer h=1024 16 heads f=4096 seq1024 x batch8
    "c2": LayerConfig("c2", 1, h=1024, f=4096, heads=16, N=8192,
                      note="GPT-2 medium layer (h=1024, ffn=4096, seq=1024, batch=8)", seq=1024),
    # c3: ViT-Large layer h=1024 16 heads 197 tokens x batch64
    "c3": LayerConfig("c3", 2, h=1024, f=4096, heads=16, N=12608,
                      note="ViT-Large layer (h=1024, 16 heads, 197 tokens, batch=64)", seq=197, causal=False),
    # c4: Llama-2-7B-shaped layer h=4096 f=11008 seq2048
    "c4": LayerConfig("c4", 3, h=4096, f=11008, heads=32, N=2048,
                      note="Llama-2-7B-shaped layer (h=4096, ffn=11008, seq=2048)", seq=2048),
    # c0 (optional, the paper's own shape): ViT-1B layer h=2048 f=8192, 65 tokens x batch 64
    "c0": LayerConfig("c0", 5, h=2048, f=8192, heads=16, N=4160,
                      note="ViT-1B layer (h=2048, ffn=8192, 65 tokens, batch=64)", seq=65, causal=False),
    # c5: GPT-13B-shaped 4-layer stack h=5120 f=20480 seq2048
    "c5": LayerConfig("c5", 4, h=5120, f=20480, heads=40, N=2048, layers=4,
                      note="GPT 13B-shaped 4-layer stack (h=5120, ffn=20480, seq=2048)", seq=2048),
}


def slowdowns(cfg: str, e: int) -> list[float]:
    """Emulated straggling skewness chi per rank."""
    chi = [1.0] * e
    if e == 1:
        return chi
    if cfg in ("c1",):
        chi[1] = 2.0
    elif cfg in ("c2", "c3"):
        chi[e - 1] = 2.0
    elif cfg == "c4":
        chi[min(5, e - 1)] = 3.0
    elif cfg == "c5":
        chi[0] = 2.0
    return chi

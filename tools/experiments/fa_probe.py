"""Probe of library attention kernels on B200 (decides NEXT-4's core): flash_attn 2 and torch SDPA backends,
fwd and fwd+bwd at the configs' attention shapes."""
import torch
from torch.nn.attention import sdpa_kernel, SDPBackend
from flash_attn import flash_attn_func
import torch.nn.functional as F


def bench(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for (B, S, H, D, causal) in [(8, 1024, 16, 64, True), (64, 197, 16, 64, False), (1, 2048, 32, 128, True)]:
    fl = 4 * B * H * S * S * D * (0.5 if causal else 1)
    q = torch.randn(B, S, H, D, device='cuda', dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn_like(q, requires_grad=True)
    v = torch.randn_like(q, requires_grad=True)
    g = torch.randn_like(q)

    def fa_f():
        return flash_attn_func(q, k, v, causal=causal)

    def fa_fb():
        flash_attn_func(q, k, v, causal=causal).backward(g)
    out = [f"{B}x{S}x{H}x{D} causal={causal}"]
    out.append("FA2 fwd %.3f ms fwd+bwd %.3f ms" % (bench(fa_f), bench(fa_fb)))
    qt, kt, vt, gt = (t.transpose(1, 2) for t in (q, k, v, g))
    for be in (SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION, SDPBackend.EFFICIENT_ATTENTION):
        try:
            with sdpa_kernel(be):
                f = bench(lambda: F.scaled_dot_product_attention(qt, kt, vt, is_causal=causal))
                fb = bench(lambda: F.scaled_dot_product_attention(qt, kt, vt, is_causal=causal).backward(gt))
            out.append(f"{be.name} fwd {f:.3f} ms ({fl / f / 1e9:.0f} TF/s) fwd+bwd {fb:.3f} ms ({3.5 * fl / fb / 1e9:.0f} TF/s)")
        except Exception as ex:
            out.append(f"{be.name} unavailable: {str(ex)[:80]}")
    print(" | ".join(out), flush=True)

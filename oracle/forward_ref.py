"""fp32 CPU Llama forward -- TEST INFRASTRUCTURE ONLY (the logit oracle).

``parity unpinned`` by the reference (it has no model code; FlashInfer is not
vendored): this is the plain-PyTorch fp32 restatement of a
Llama-2 prefill over the same bf16 weights the GPU runs (HF Llama semantics:
RMSNorm, rotate-half RoPE with theta 1e4, causal softmax attention, SiLU-gated
MLP, untied lm_head).  A ZigZag split ``(T_i, S_i)`` (livescale.py:4-14,
PAPER.md:585-589) runs the same function on two instances, so cooperative
logits are compared with this unsplit forward: max relative error <= 1e-2 and
identical greedy tokens (north star).
"""

from __future__ import annotations

import math

import torch


def _rmsnorm(x, w, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w


def _rope(x, pos, theta):
    # x [B, S, H, hd]
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-(torch.arange(0, half, dtype=torch.float64) * 2.0) / hd)
    ang = pos.to(torch.float64)[:, None] * inv[None, :]
    cos, sin = ang.cos().float(), ang.sin().float()
    cos = cos[None, :, None, :]
    sin = sin[None, :, None, :]
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)


def _bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).float()


def block_fp32(arch, w: dict, x: torch.Tensor, bf16_storage: bool = False) -> torch.Tensor:
    """One Llama block in fp32. x [B, S, d]; w: fp32 CPU tensors.

    ``bf16_storage``: round every intermediate the GPU path stores in bf16 (norm
    outputs, the fused q/k/v projection before and after RoPE, the attention
    output, the residual stream after each sub-layer, gate/up, the SiLU product)
    -- the same computation at the GPU's storage precision, math still fp32.
    It measures the bf16 floor: what ANY bf16-activation implementation loses
    against the fp32 forward on the same inputs."""
    r = _bf16 if bf16_storage else (lambda t: t)
    B, S, d = x.shape
    H, KV, hd = arch.n_heads, arch.n_kv_heads, arch.head_dim
    h = r(_rmsnorm(x, w["attn_norm"], arch.norm_eps))
    qkv = r(h @ w["wqkv"].t())
    q = qkv[..., : H * hd].view(B, S, H, hd)
    k = qkv[..., H * hd:(H + KV) * hd].view(B, S, KV, hd)
    v = qkv[..., (H + KV) * hd:].view(B, S, KV, hd)
    pos = torch.arange(S)
    q, k = r(_rope(q, pos, arch.rope_theta)), r(_rope(k, pos, arch.rope_theta))
    if KV != H:
        k = k.repeat_interleave(H // KV, dim=2)
        v = v.repeat_interleave(H // KV, dim=2)
    q, k, v = (t.transpose(1, 2) for t in (q, k, v))
    scores = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    mask = torch.ones(S, S, dtype=torch.bool).triu(1)
    scores = scores.masked_fill(mask, float("-inf"))
    att = r(torch.softmax(scores, dim=-1) @ v)
    o = r(x + att.transpose(1, 2).reshape(B, S, H * hd) @ w["wo"].t())
    h2 = r(_rmsnorm(o, w["ffn_norm"], arch.norm_eps))
    gu = r(h2 @ w["wgu"].t())
    g, u = gu[..., : arch.ffn], gu[..., arch.ffn:]
    return r(o + r(torch.nn.functional.silu(g) * u) @ w["wdown"].t())


def forward_fp32(arch, layers: list[dict], tokens: torch.Tensor, bf16_storage: bool = False) -> torch.Tensor:
    """Unsplit prefill -> logits of each sequence's last token, fp32 [B, vocab].
    ``bf16_storage`` as in ``block_fp32`` (the head stays fp32, as on the GPU)."""
    x = layers[0]["embed"][tokens]
    for w in layers:
        x = block_fp32(arch, w, x, bf16_storage)
    last = _rmsnorm(x[:, -1], layers[-1]["final_norm"], arch.norm_eps)
    if bf16_storage:
        last = _bf16(last)
    return last @ layers[-1]["lm_head"].t()


def weights_to_cpu_fp32(slab_weights) -> list[dict]:
    return [{k: v.detach().float().cpu() for k, v in layer.items()} for layer in slab_weights.layers]

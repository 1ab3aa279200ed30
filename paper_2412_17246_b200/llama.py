"""Llama forward over weights that live in a layer slab (cooperative execution body).

The reference has no model code: a batch's prefill is ``alpha + beta*tokens``
milliseconds (parampool.py:58-62) and a live pair serves at
``max(k, L-k)/L`` of that (simcore.py:408-417).  Here the layers really run:
each load unit of the slab (slab.py) is viewed in place as the block's
tensors, so a target GPU can execute block ``k`` the moment the tracker
publishes unit ``k`` -- no copy out of the landing slab.

Per block (all bf16, fp32 accumulation):
  h   = rmsnorm(x)                 bz_rmsnorm
  qkv = h . Wqkv^T                 bz_gemm_bf16 (tcgen05)
  rope(q, k)                       bz_rope
  a   = causal attention(q, k, v)  torch SDPA (library kernel, like cuBLAS)
  o   = a . Wo^T + x               bz_gemm_bf16 with residual epilogue
  g   = rmsnorm(o) . Wgu^T         bz_rmsnorm + bz_gemm_bf16
  x'  = silu(g1)*g2 . Wdown^T + o  bz_silu_mul + bz_gemm_bf16 residual epilogue

Unit byte layout (tensor order inside a unit, each [out, in] row-major):
  [embed vocab x d]   (unit 1 only)
  attn_norm d | Wqkv (d + 2 kv) x d | Wo d x d | ffn_norm d | Wgu 2 ffn x d | Wdown d x ffn
  [final_norm d | lm_head vocab x d]   (unit L only)
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import torch

from ._native import cuda_lib
from .slab import LlamaArch, SlabLayout


def _entries(arch: LlamaArch, k: int) -> list[tuple[str, tuple[int, ...]]]:
    d, kv, ffn, v = arch.d_model, arch.kv_dim, arch.ffn, arch.vocab
    out = []
    if k == 0:
        out.append(("embed", (v, d)))
    out += [("attn_norm", (d,)), ("wqkv", (d + 2 * kv, d)), ("wo", (d, d)), ("ffn_norm", (d,)),
            ("wgu", (2 * ffn, d)), ("wdown", (d, ffn))]
    if k == arch.n_layers - 1:
        out += [("final_norm", (d,)), ("lm_head", (v, d))]
    return out


class SlabWeights:
    """bf16 tensor views of every block's weights inside a slab's data region."""

    def __init__(self, arch: LlamaArch, layout: SlabLayout, data: torch.Tensor):
        if data.dtype != torch.uint8:
            raise TypeError("slab data must be a uint8 view")
        if arch.d_model % 128:
            raise ValueError("d_model must be a multiple of 128 (256-byte tensor alignment)")
        self.arch = arch
        self.layout = layout
        self.layers: list[dict[str, torch.Tensor]] = []
        for k in range(arch.n_layers):
            off = layout.unit_off[k]
            views = {}
            for name, shape in _entries(arch, k):
                n = 1
                for s in shape:
                    n *= s
                views[name] = data[off:off + 2 * n].view(torch.bfloat16).view(*shape)
                off += 2 * n
            if off - layout.unit_off[k] != layout.unit_bytes[k]:
                raise ValueError(f"unit {k} size mismatch: {off - layout.unit_off[k]} vs {layout.unit_bytes[k]}")
            self.layers.append(views)

    @torch.no_grad()
    def init_random(self, seed: int = 0, std: float = 0.02):
        """Synthetic random-init weights (no checkpoints offline): N(0, std) matrices,
        unit-ish norms.  Deterministic on a given device."""
        g = torch.Generator(device=self.layers[0]["wqkv"].device)
        g.manual_seed(seed)
        for views in self.layers:
            for name, t in views.items():
                if name.endswith("norm"):
                    t.copy_(1.0 + 0.1 * torch.randn(t.shape, generator=g, device=t.device))
                else:
                    t.copy_(std * torch.randn(t.shape, generator=g, device=t.device))


@dataclass
class Batch:
    """B equal-length sequences of S tokens (prefill)."""

    tokens: torch.Tensor      # int64 [B, S]

    @property
    def shape(self):
        return tuple(self.tokens.shape)


class LlamaExecutor:
    """Runs blocks of a slab-resident Llama on this GPU with the libblitz kernels."""

    def __init__(self, weights: SlabWeights, max_tokens: int, device):
        self.w = weights
        self.arch = weights.arch
        self.lib = cuda_lib()
        a = self.arch
        dev = torch.device(device)
        bf = torch.bfloat16
        self.h = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.qkv = torch.empty(max_tokens, a.d_model + 2 * a.kv_dim, dtype=bf, device=dev)
        self.attn = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.o = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.gu = torch.empty(max_tokens, 2 * a.ffn, dtype=bf, device=dev)
        self.act = torch.empty(max_tokens, a.ffn, dtype=bf, device=dev)
        self.max_tokens = max_tokens

    def _gemm(self, x, w, out, residual=None):
        m, k = x.shape
        n = w.shape[0]
        self.lib.bz_gemm_bf16(x.data_ptr(), w.data_ptr(), out.data_ptr(),
                              residual.data_ptr() if residual is not None else None,
                              m, n, k, x.stride(0), w.stride(0), out.stride(0),
                              residual.stride(0) if residual is not None else 0, 0,
                              torch.cuda.current_stream().cuda_stream)
        return out

    def _rmsnorm(self, x, w, out):
        self.lib.bz_rmsnorm(x.data_ptr(), w.data_ptr(), out.data_ptr(), x.shape[0], x.shape[1],
                            x.stride(0), out.stride(0), self.arch.norm_eps,
                            torch.cuda.current_stream().cuda_stream)
        return out

    def embed(self, tokens: torch.Tensor) -> torch.Tensor:
        return self.w.layers[0]["embed"].index_select(0, tokens.reshape(-1)).contiguous()

    @torch.no_grad()
    def block(self, k: int, x: torch.Tensor, positions: torch.Tensor, bs: tuple[int, int],
              out: Optional[torch.Tensor] = None, signal: Optional[torch.Tensor] = None) -> torch.Tensor:
        """x [B*S, d] -> block k output; positions int32 [B*S].

        ``out`` may live on another GPU (peer access): the down-projection GEMM
        then stores the block output straight into it over NVLink and, with
        ``signal``, raises that u32 counter by its CTA count when done (the fused
        hand-off of cooperative execution).  Returns ``out`` (or a new tensor).
        """
        a, L = self.arch, self.w.layers[k]
        m = x.shape[0]
        B, S = bs
        s = torch.cuda.current_stream().cuda_stream
        h, qkv, attn, o = self.h[:m], self.qkv[:m], self.attn[:m], self.o[:m]
        self._rmsnorm(x, L["attn_norm"], h)
        self._gemm(h, L["wqkv"], qkv)
        self.lib.bz_rope(qkv.data_ptr(), positions.data_ptr(), m, a.n_heads + a.n_kv_heads,
                         a.head_dim, qkv.stride(0), a.rope_theta, s)
        hd, H, KV = a.head_dim, a.n_heads, a.n_kv_heads
        q = qkv[:, : H * hd].view(B, S, H, hd).transpose(1, 2)
        kk = qkv[:, H * hd:(H + KV) * hd].view(B, S, KV, hd).transpose(1, 2)
        v = qkv[:, (H + KV) * hd:].view(B, S, KV, hd).transpose(1, 2)
        att = torch.nn.functional.scaled_dot_product_attention(q, kk, v, is_causal=True,
                                                               enable_gqa=KV != H)
        attn.copy_(att.transpose(1, 2).reshape(m, H * hd))
        self._gemm(attn, L["wo"], o, residual=x)
        self._rmsnorm(o, L["ffn_norm"], h)
        gu, act = self.gu[:m], self.act[:m]
        self._gemm(h, L["wgu"], gu)
        self.lib.bz_silu_mul(gu.data_ptr(), act.data_ptr(), m, a.ffn, gu.stride(0), act.stride(0), s)
        if out is None:
            out = torch.empty_like(x)
        if signal is None:
            self._gemm(act, L["wdown"], out, residual=o)
            self.last_signal_ctas = 0
        else:
            import ctypes
            ctas = ctypes.c_int(0)
            w = L["wdown"]
            self.lib.bz_gemm_bf16_signal(act.data_ptr(), w.data_ptr(), out.data_ptr(), o.data_ptr(),
                                         m, w.shape[0], act.shape[1], act.stride(0), w.stride(0),
                                         out.stride(0), o.stride(0), 0, signal.data_ptr(),
                                         ctypes.byref(ctas), s)
            self.last_signal_ctas = ctas.value
        return out

    @torch.no_grad()
    def head(self, x: torch.Tensor, bs: tuple[int, int]) -> torch.Tensor:
        """Final norm + lm_head on each sequence's last token -> fp32 logits [B, vocab]."""
        B, S = bs
        last = x.view(B, S, -1)[:, -1].contiguous()
        L = self.w.layers[-1]
        h = torch.empty_like(last)
        self._rmsnorm(last, L["final_norm"], h)
        logits = torch.empty(B, self.arch.vocab, dtype=torch.bfloat16, device=x.device)
        self._gemm(h, L["lm_head"], logits)
        return logits.float()

    @torch.no_grad()
    def forward(self, tokens: torch.Tensor, first: int = 0, last: Optional[int] = None,
                x: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Blocks [first, last) (0-based); returns hidden, or logits if last == L."""
        B, S = tokens.shape
        last = self.arch.n_layers if last is None else last
        pos = torch.arange(S, dtype=torch.int32, device=tokens.device).repeat(B)
        if x is None:
            x = self.embed(tokens)
        for k in range(first, last):
            x = self.block(k, x, pos, (B, S))
        return self.head(x, (B, S)) if last == self.arch.n_layers else x

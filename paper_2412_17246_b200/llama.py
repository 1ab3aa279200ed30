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
  a   = causal attention(q, k, v)  bz_prefill_attention (tcgen05 flash kernel, writes [tokens, H*hd])
  o   = a . Wo^T + x               bz_gemm_bf16 with residual epilogue
  g   = rmsnorm(o) . Wgu^T         bz_rmsnorm + bz_gemm_bf16
  x'  = silu(g1)*g2 . Wdown^T + o  bz_silu_mul + bz_gemm_bf16 residual epilogue

Unit byte layout (tensor order inside a unit, each [out, in] row-major):
  [embed vocab x d]   (unit 1 only)
  attn_norm d | Wqkv (d + 2 kv) x d | Wo d x d | ffn_norm d | Wgu 2 ffn x d | Wdown d x ffn
  [final_norm d | lm_head vocab x d]   (unit L only)
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import torch

from ._native import BZ_GEMM_B_STATIC, BZ_GEMM_C_F32, BzDecodeBlock, cuda_lib
from .slab import LlamaArch, SlabLayout


# prefill attention: the tcgen05 flash kernel (csrc/attention_tcgen05.cu, 0.89-1.08x of
# cuDNN's kernel on the 7B shapes, ahead at batch 1; profiles/r2_attn_bench_v5.jsonl);
# BZ_PREFILL_ATTN=sdpa runs torch SDPA instead for A/B measurements
PREFILL_ATTENTION = os.environ.get("BZ_PREFILL_ATTN", "tcgen05")

# small-batch decode: one persistent kernel per decode step (csrc/decode_fused.cu) for
# 1..FUSED_MAX_ROWS sequences.  Opt-in (BZ_DECODE_FUSED=1): on B200 it measured 103.6 vs
# 106.0 us per 7B block at batch 1 and slower at 2..4 rows (its attention items and
# per-row staging are latency-bound), profiles/r2_fused_decode.txt
FUSED_DECODE = os.environ.get("BZ_DECODE_FUSED", "0") == "1"
FUSED_MAX_ROWS = 4


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
        dev = torch.device(device)
        self.lib = cuda_lib(dev.index if dev.index is not None else torch.cuda.current_device())
        a = self.arch
        bf = torch.bfloat16
        self.h = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.qkv = torch.empty(max_tokens, a.d_model + 2 * a.kv_dim, dtype=bf, device=dev)
        self.attn = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.o = torch.empty(max_tokens, a.d_model, dtype=bf, device=dev)
        self.gu = torch.empty(max_tokens, 2 * a.ffn, dtype=bf, device=dev)
        self.act = torch.empty(max_tokens, a.ffn, dtype=bf, device=dev)
        self.max_tokens = max_tokens
        # stream-K counters + fp32 partials for skinny (decode) GEMMs; one executor = one stream
        self.streamk_ws = torch.zeros(self.STREAMK_WS_BYTES // 4, dtype=torch.float32, device=dev)
        self.last_signal_ctas = 0
        self._attn_ws: Optional[torch.Tensor] = None   # V^T of the prefill attention (grown on demand)

    STREAMK_WS_BYTES = 64 << 20

    def _gemm(self, x, w, out, residual=None, signal=None):
        import ctypes
        m, k = x.shape
        n = w.shape[0]
        ctas = ctypes.c_int(0)
        # B = slab weights: landed before the layer gate; an fp32 out keeps the accumulator
        flags = BZ_GEMM_B_STATIC | (BZ_GEMM_C_F32 if out.dtype == torch.float32 else 0)
        self.lib.bz_gemm_bf16_ex(x.data_ptr(), w.data_ptr(), out.data_ptr(),
                                 residual.data_ptr() if residual is not None else None,
                                 m, n, k, x.stride(0), w.stride(0), out.stride(0),
                                 residual.stride(0) if residual is not None else 0, 0,
                                 flags,
                                 self.streamk_ws.data_ptr(), self.STREAMK_WS_BYTES,
                                 signal.data_ptr() if signal is not None else None, ctypes.byref(ctas),
                                 torch.cuda.current_stream().cuda_stream)
        self.last_signal_ctas = ctas.value if signal is not None else 0
        return out

    def _rmsnorm(self, x, w, out):
        self.lib.bz_rmsnorm(x.data_ptr(), w.data_ptr(), out.data_ptr(), x.shape[0], x.shape[1],
                            x.stride(0), out.stride(0), self.arch.norm_eps,
                            torch.cuda.current_stream().cuda_stream)
        return out

    def embed(self, tokens: torch.Tensor) -> torch.Tensor:
        table = self.w.layers[0]["embed"]
        return table.index_select(0, tokens.reshape(-1).to(table.device, non_blocking=True)).contiguous()

    def _attn_in(self, k: int, x: torch.Tensor, positions: torch.Tensor):
        """rmsnorm -> qkv GEMM -> rope; returns q, k, v as [rows, heads, hd] views."""
        a, L = self.arch, self.w.layers[k]
        m = x.shape[0]
        h, qkv = self.h[:m], self.qkv[:m]
        self._rmsnorm(x, L["attn_norm"], h)
        self._gemm(h, L["wqkv"], qkv)
        self.lib.bz_rope(qkv.data_ptr(), positions.data_ptr(), m, a.n_heads + a.n_kv_heads,
                         a.head_dim, qkv.stride(0), a.rope_theta, torch.cuda.current_stream().cuda_stream)
        hd, H, KV = a.head_dim, a.n_heads, a.n_kv_heads
        return (qkv[:, : H * hd].view(m, H, hd), qkv[:, H * hd:(H + KV) * hd].view(m, KV, hd),
                qkv[:, (H + KV) * hd:].view(m, KV, hd))

    def _attn_out_mlp(self, k: int, x: torch.Tensor, attn: torch.Tensor,
                      out: Optional[torch.Tensor], signal: Optional[torch.Tensor]) -> torch.Tensor:
        """o = attn . Wo^T + x; out = o + mlp(rmsnorm(o)) (optionally fused hand-off)."""
        a, L = self.arch, self.w.layers[k]
        m = x.shape[0]
        s = torch.cuda.current_stream().cuda_stream
        h, o, gu, act = self.h[:m], self.o[:m], self.gu[:m], self.act[:m]
        self._gemm(attn, L["wo"], o, residual=x)
        self._rmsnorm(o, L["ffn_norm"], h)
        self._gemm(h, L["wgu"], gu)
        self.lib.bz_silu_mul(gu.data_ptr(), act.data_ptr(), m, a.ffn, gu.stride(0), act.stride(0), s)
        if out is None:
            out = torch.empty_like(x)
        return self._gemm(act, L["wdown"], out, residual=o, signal=signal)

    @torch.no_grad()
    def block(self, k: int, x: torch.Tensor, positions: torch.Tensor, bs: tuple[int, int],
              out: Optional[torch.Tensor] = None, signal: Optional[torch.Tensor] = None,
              kv: Optional["KVCache"] = None) -> torch.Tensor:
        """Prefill of block k: x [B*S, d] -> block output; positions int32 [B*S].

        ``out`` may live on another GPU (peer access): the down-projection GEMM
        then stores the block output straight into it over NVLink and, with
        ``signal``, raises that u32 counter by its CTA count when done (the fused
        hand-off of cooperative execution).  With ``kv`` the block's keys and
        values land in the cache (positions 0..S-1) for later decode steps.
        Returns ``out`` (or a new tensor).
        """
        a = self.arch
        m = x.shape[0]
        B, S = bs
        H, KV, hd = a.n_heads, a.n_kv_heads, a.head_dim
        q, kk, v = (t.view(B, S, -1, hd).transpose(1, 2) for t in self._attn_in(k, x, positions))
        if kv is not None:
            kv.store_prefill(k, kk, v)
        attn = self.attn[:m]
        if PREFILL_ATTENTION == "tcgen05":
            self._prefill_attention(B, S, attn)
        else:
            att = torch.nn.functional.scaled_dot_product_attention(q, kk, v, is_causal=True,
                                                                   enable_gqa=KV != H)
            attn.copy_(att.transpose(1, 2).reshape(m, H * hd))
        return self._attn_out_mlp(k, x, attn, out, signal)

    def _prefill_attention(self, B: int, S: int, attn: torch.Tensor):
        """Causal attention of the roped qkv rows into ``attn`` [B*S, H*hd]: the tcgen05
        flash kernel (csrc/attention_tcgen05.cu), V transposed into a workspace."""
        import ctypes
        a = self.arch
        need = ctypes.c_int64()
        self.lib.bz_prefill_attention_workspace_bytes(B, S, a.n_kv_heads, a.head_dim, ctypes.byref(need))
        if self._attn_ws is None or self._attn_ws.numel() < need.value:
            self._attn_ws = torch.empty(need.value, dtype=torch.uint8, device=self.h.device)
        qkv = self.qkv[:B * S]
        self.lib.bz_prefill_attention(qkv.data_ptr(), qkv.stride(0), B, S, a.n_heads, a.n_kv_heads, a.head_dim,
                                      self._attn_ws.data_ptr(), self._attn_ws.numel(), attn.data_ptr(),
                                      attn.stride(0), torch.cuda.current_stream().cuda_stream)

    @torch.no_grad()
    def decode_block(self, k: int, x: torch.Tensor, kv: "KVCache",
                     out: Optional[torch.Tensor] = None, signal: Optional[torch.Tensor] = None) -> torch.Tensor:
        """One decode step of block k for B sequences: x [B, d] is the hidden state
        of each sequence's newest token, at the cache's device position.  Its key/
        value are appended (bz_rope_append) and it attends over positions 0..pos
        (bz_decode_attention) -- no host-side position, so the step is graph-safe."""
        kv.require_room()
        a, L = self.arch, self.w.layers[k]
        B = x.shape[0]
        s = torch.cuda.current_stream().cuda_stream
        h, qkv, attn = self.h[:B], self.qkv[:B], self.attn[:B]
        self._rmsnorm(x, L["attn_norm"], h)
        self._gemm(h, L["wqkv"], qkv)
        kc, vc = kv.k[k], kv.v[k]
        # one device position for the batch, or one per row (continuous batching)
        rope = self.lib.bz_rope_append_rows if kv.per_row else self.lib.bz_rope_append
        attend = self.lib.bz_decode_attention_rows if kv.per_row else self.lib.bz_decode_attention
        rope(qkv.data_ptr(), qkv.stride(0), B, a.n_heads, a.n_kv_heads, a.head_dim, a.rope_theta, kc.data_ptr(),
             vc.data_ptr(), kv.max_seq, kv.pos_dev.data_ptr(), s)
        attend(qkv.data_ptr(), qkv.stride(0), kc.data_ptr(), vc.data_ptr(), B, a.n_heads, a.n_kv_heads, a.head_dim,
               kv.max_seq, kv.pos_dev.data_ptr(), attn.data_ptr(), attn.stride(0), kv.workspace.data_ptr(),
               kv.workspace.numel(), s)
        return self._attn_out_mlp(k, x, attn, out, signal)

    def fused_decode_ok(self, rows: int, kv: "KVCache", first: int, last: int) -> bool:
        """Whether bz_decode_fused covers this step (shapes its kernel supports)."""
        a = self.arch
        return (FUSED_DECODE and 1 <= rows <= FUSED_MAX_ROWS and a.head_dim in (64, 128)
                and a.n_heads % a.n_kv_heads == 0 and a.n_heads // a.n_kv_heads <= 8
                and a.d_model == a.n_heads * a.head_dim and a.d_model % 64 == 0 and a.ffn % 64 == 0
                and 0 < kv.max_seq <= 131072 and last > first)

    def decode_blocks(self, first: int, last: int, x: torch.Tensor, kv: "KVCache") -> torch.Tensor:
        """Blocks [first, last) of one decode step for x [B, d]: one bz_decode_fused launch
        for 1..4 sequences, else decode_block per block.  Returns a new [B, d] tensor."""
        kv.require_room()
        B = x.shape[0]
        if not self.fused_decode_ok(B, kv, first, last):
            for k in range(first, last):
                x = self.decode_block(k, x, kv)
            return x
        a = self.arch
        out = x.contiguous().clone()   # updated in place by the kernel
        ws = self._fused_workspace(B)
        self.lib.bz_decode_fused(self._fused_blocks(kv, first, last), last - first, out.data_ptr(), out.stride(0), B,
                                 a.d_model, a.n_heads, a.n_kv_heads, a.head_dim, a.ffn, a.rope_theta, a.norm_eps,
                                 kv.max_seq, kv.pos_dev.data_ptr(), 1 if kv.per_row else 0, ws.data_ptr(),
                                 ws.numel(), 0, torch.cuda.current_stream().cuda_stream)
        return out

    def _fused_workspace(self, rows: int) -> torch.Tensor:
        import ctypes
        cache = self.__dict__.setdefault("_fused_ws", {})
        if rows not in cache:
            a = self.arch
            nb = ctypes.c_int64(0)
            self.lib.bz_decode_fused_workspace_bytes(rows, a.d_model, a.n_heads, a.n_kv_heads, a.head_dim, a.ffn,
                                                     ctypes.byref(nb))
            cache[rows] = torch.zeros(nb.value, dtype=torch.uint8, device=self.h.device)  # zeroed once
        return cache[rows]

    def _fused_blocks(self, kv: "KVCache", first: int, last: int):
        """The bz_decode_block array of blocks [first, last) against this cache (kept on the
        cache, so it lives exactly as long as the panels it points into)."""
        cache = kv.__dict__.setdefault("_fused_blocks", {})
        key = (id(self), first, last)
        if key not in cache:
            arr = (BzDecodeBlock * (last - first))()
            for i, k in enumerate(range(first, last)):
                L = self.w.layers[k]
                arr[i] = BzDecodeBlock(L["attn_norm"].data_ptr(), L["wqkv"].data_ptr(), L["wo"].data_ptr(),
                                       L["ffn_norm"].data_ptr(), L["wgu"].data_ptr(), L["wdown"].data_ptr(),
                                       kv.k[k].data_ptr(), kv.v[k].data_ptr())
            cache[key] = arr
        return cache[key]

    def fused_decode_timed_out(self, rows: int) -> bool:
        """True if the last fused decode step of this batch size hit its grid-barrier timeout."""
        import ctypes
        flag = ctypes.c_int(0)
        self.lib.bz_decode_fused_status(self._fused_workspace(rows).data_ptr(), ctypes.byref(flag),
                                        torch.cuda.current_stream().cuda_stream)
        return bool(flag.value)

    @torch.no_grad()
    def head(self, x: torch.Tensor, bs: tuple[int, int]) -> torch.Tensor:
        """Final norm + lm_head on each sequence's last token -> fp32 logits [B, vocab]."""
        B, S = bs
        last = x.view(B, S, -1)[:, -1].contiguous()
        L = self.w.layers[-1]
        h = torch.empty_like(last)
        self._rmsnorm(last, L["final_norm"], h)
        # fp32 logits straight from the TMEM accumulator (no bf16 rounding of the head)
        logits = torch.empty(B, self.arch.vocab, dtype=torch.float32, device=x.device)
        self._gemm(h, L["lm_head"], logits)
        return logits

    @torch.no_grad()
    def forward(self, tokens: torch.Tensor, first: int = 0, last: Optional[int] = None,
                x: Optional[torch.Tensor] = None, kv: Optional["KVCache"] = None) -> torch.Tensor:
        """Prefill blocks [first, last) (0-based); returns hidden, or logits if last == L.
        With ``kv`` (covering those blocks) the prompt's keys/values are cached and
        ``kv.length`` becomes S."""
        B, S = tokens.shape
        last = self.arch.n_layers if last is None else last
        pos = torch.arange(S, dtype=torch.int32, device=tokens.device).repeat(B)
        if x is None:
            x = self.embed(tokens)
        for k in range(first, last):
            x = self.block(k, x, pos, (B, S), kv=kv)
        if kv is not None:
            kv.length = S
        return self.head(x, (B, S)) if last == self.arch.n_layers else x

    @torch.no_grad()
    def decode(self, tokens: torch.Tensor, kv: "KVCache", first: int = 0, last: Optional[int] = None,
               x: Optional[torch.Tensor] = None) -> torch.Tensor:
        """One decode step over blocks [first, last) for the newest token of each
        sequence (tokens int64 [B]); returns hidden [B, d], or fp32 logits [B, vocab]
        if last == L.  Advances ``kv.length`` by one."""
        kv.require_room()  # before anything is enqueued: a full cache must not be written
        last = self.arch.n_layers if last is None else last
        if x is None:
            x = self.embed(tokens)
        x = self.decode_blocks(first, last, x, kv)
        kv.advance()
        return self.head(x, (x.shape[0], 1)) if last == self.arch.n_layers else x

    def decode_graph(self, kv: "KVCache", first: int = 0, last: Optional[int] = None,
                     hidden_in: bool = False, head: Optional[bool] = None) -> "DecodeGraph":
        last = self.arch.n_layers if last is None else last
        return DecodeGraph(self, kv, first, last, hidden_in, last == self.arch.n_layers if head is None else head)


class KVCache:
    """Keys/values of B equal-length sequences for blocks [first, last) on one GPU,
    each ``[B, KV, max_seq, hd]`` bf16 (one contiguous [max_seq, hd] panel per
    sequence and kv head).  Under a ZigZag split the target holds blocks
    [0, T_i) and the source [T_i, L) of batch i -- exactly where the prefill ran
    them -- so decode continues with the same split and moves only the [B, d]
    hand-off.

    The next write position lives on the device (``pos_dev``) and is advanced by
    the decode step itself, so a captured step replays at every position; the
    host mirror ``length`` is kept in step by ``advance``.
    """

    def __init__(self, arch: LlamaArch, batch: int, max_seq: int, device, first: int = 0,
                 last: Optional[int] = None, per_row: bool = False):
        from ._native import cuda_lib
        import ctypes

        last = arch.n_layers if last is None else last
        shape = (batch, arch.n_kv_heads, max_seq, arch.head_dim)
        self.k = {l: torch.zeros(shape, dtype=torch.bfloat16, device=device) for l in range(first, last)}
        self.v = {l: torch.zeros(shape, dtype=torch.bfloat16, device=device) for l in range(first, last)}
        self.batch, self.max_seq = batch, max_seq
        # per_row: every row (sequence slot) has its own device position -- continuous
        # batching; ``length`` then tracks nothing (slots are managed by the caller)
        self.per_row = per_row
        self.pos_dev = torch.zeros(batch if per_row else 1, dtype=torch.int32, device=device)
        nbytes = ctypes.c_int64(0)
        cuda_lib().bz_decode_workspace_bytes(batch, arch.n_heads, arch.n_kv_heads, arch.head_dim, max_seq,
                                             ctypes.byref(nbytes))
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=device)
        self._arch_heads = arch.n_heads
        self._length = 0

    @property
    def length(self) -> int:
        return self._length

    @length.setter
    def length(self, n: int):
        if not 0 <= n <= self.max_seq:
            raise ValueError("cache length out of range")
        self._length = n
        self.pos_dev.fill_(n)

    def require_room(self):
        """Raise before a decode step is enqueued if the cache has no free position
        (the device kernels also refuse to write past a panel).  Per-row caches are
        managed slot by slot by their caller; the device guard protects them."""
        if self.per_row:
            return
        if self._length >= self.max_seq:
            raise ValueError(f"KV cache full ({self._length} of {self.max_seq} positions)")

    def advance(self):
        """After a decode step: the device position moves on the current stream."""
        self.require_room()
        self._length += 1
        self.pos_dev.add_(1)

    def rows_view(self, n: int) -> "KVCache":
        """The first ``n`` rows (sequence slots) of a per-row cache as a cache of batch n
        sharing its storage and positions (a decode graph per batch-size bucket)."""
        if not self.per_row or not 0 < n <= self.batch:
            raise ValueError("rows_view needs a per-row cache and 0 < n <= batch")
        v = object.__new__(KVCache)
        v.k = {l: t[:n] for l, t in self.k.items()}
        v.v = {l: t[:n] for l, t in self.v.items()}
        v.batch, v.max_seq, v.per_row = n, self.max_seq, True
        v.pos_dev = self.pos_dev[:n]
        import ctypes
        from ._native import cuda_lib
        nb = ctypes.c_int64(0)
        first = next(iter(self.k.values()))
        cuda_lib().bz_decode_workspace_bytes(n, self._arch_heads, first.shape[1], first.shape[3], self.max_seq,
                                             ctypes.byref(nb))
        v.workspace = torch.empty(nb.value, dtype=torch.uint8, device=first.device)
        v._arch_heads = self._arch_heads
        v._length = 0
        return v

    def bytes(self) -> int:
        return sum(t.numel() * 2 for t in list(self.k.values()) + list(self.v.values()))

    def store_prefill(self, layer: int, k: torch.Tensor, v: torch.Tensor):
        s = k.shape[2]
        if s > self.max_seq:
            raise ValueError("prompt longer than the cache")
        self.k[layer][:, :, :s].copy_(k)
        self.v[layer][:, :, :s].copy_(v)


class DecodeGraph:
    """A whole decode step (blocks [first, last), plus the head when last == L)
    captured once as a CUDA graph and replayed per token: the position comes
    from ``kv.pos_dev``, so there is no host work per step beyond the replay.
    ``hidden_in`` feeds a [B, d] hidden state instead of token ids (the source
    side of a cooperative split)."""

    def __init__(self, ex: "LlamaExecutor", kv: KVCache, first: int, last: int, hidden_in: bool = False,
                 head: bool = True):
        self.ex, self.kv, self.first, self.last, self.with_head = ex, kv, first, last, head
        dev = ex.h.device
        B = kv.batch
        self.tokens = torch.zeros(B, dtype=torch.int64, device=dev)
        self.hidden = torch.zeros(B, ex.arch.d_model, dtype=torch.bfloat16, device=dev) if hidden_in else None
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        saved = kv.length
        saved_pos = kv.pos_dev.clone() if kv.per_row else None
        with torch.cuda.stream(side):
            # warm-up outside capture (lazy library init); writes position `saved`,
            # which the first real step overwrites before attending to it
            self._body()
            if kv.per_row:
                kv.pos_dev.copy_(saved_pos)
            else:
                kv.length = saved
            side.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=side):
                self.out = self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        kv._length = saved

    def _body(self):
        ex, kv = self.ex, self.kv
        x = self.hidden if self.hidden is not None else ex.embed(self.tokens)
        x = ex.decode_blocks(self.first, self.last, x, kv)
        kv.pos_dev.add_(1)
        if self.with_head:
            return ex.head(x, (x.shape[0], 1))
        return x

    def __call__(self, tokens: Optional[torch.Tensor] = None, hidden: Optional[torch.Tensor] = None):
        if not self.kv.per_row and self.kv.length >= self.kv.max_seq:
            raise ValueError("KV cache full")
        if tokens is not None:
            self.tokens.copy_(tokens)
        if hidden is not None:
            self.hidden.copy_(hidden)
        self.graph.replay()
        if not self.kv.per_row:
            self.kv._length += 1
        return self.out

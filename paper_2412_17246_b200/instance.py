"""A slab-backed serving instance: the object the reference's role mutation flips.

Reference: ``mutate_prefill_to_decode`` / ``mutate_decode_to_prefill``
(livescale.py:512-544) flip ``instance.role`` after checking it is a prefill
instance that is not mid-scale and has every layer resident; the simulator
calls it when decode runs short (simcore.py:628-653) and counts the flip as a
zero-transfer scale.  There the instance is a bookkeeping record.  Here it is
a real engine on one B200: its parameters are a layer slab (slab.py), its
``loaded_layers`` is the slab's device readiness counter (the tracker K4 writes
it), and after a flip the same slab and the prompts' KV caches serve decode
steps -- no bytes move, which tests assert by pointer identity.

The mutation functions themselves are the mirrored reference ones
(``livescale.mutate_prefill_to_decode``); this class only provides the
attributes they read (``role``, ``live_session``, ``loaded_layers``,
``total_layers``, ``model_name``).
"""

from __future__ import annotations

from typing import Optional

import torch

from .livescale import ProtocolError
from .llama import KVCache, LlamaExecutor, SlabWeights
from .slab import LlamaArch


class ServingInstance:
    ROLES = ("prefill", "decode", "colocated")

    def __init__(self, name: str, arch: LlamaArch, slab, role: str = "prefill", max_tokens: int = 4096,
                 device: Optional[int] = None):
        if role not in self.ROLES:
            raise ValueError(f"unknown role {role!r}")
        self.name = name
        self.arch = arch
        self.model_name = arch.name
        self.slab = slab
        self.role = role
        self.live_session = None          # set while a live scale targets this instance
        self.weights = SlabWeights(arch, slab.layout, slab.data)
        dev = slab.data.device if device is None else torch.device("cuda", device)
        self.executor = LlamaExecutor(self.weights, max_tokens=max_tokens, device=dev)

    # ---- attributes read by mutate_prefill_to_decode (livescale.py:512-536) -------------
    @property
    def total_layers(self) -> int:
        return self.arch.n_layers

    @property
    def loaded_layers(self) -> int:
        """Layers the device tracker has published for this slab (host read of the
        device counter; a fully written source slab is marked by ``mark_resident``)."""
        return int(self.slab.loaded.item())

    def mark_resident(self):
        """A source whose weights were written in place (init / checkpoint load)."""
        self.slab.loaded.fill_(self.arch.n_layers)

    # ---- serving ---------------------------------------------------------------------------
    def _require(self, *roles):
        if self.role not in roles:
            raise ProtocolError(f"{self.name} is a {self.role} instance")
        if self.loaded_layers < self.total_layers:
            raise ProtocolError(f"{self.name}: parameters not fully resident")

    @torch.no_grad()
    def prefill(self, tokens: torch.Tensor, max_new_tokens: int = 0) -> tuple[torch.Tensor, KVCache]:
        """Prompt pass (tokens int64 [B, S]) -> (fp32 last-token logits [B, vocab],
        the KV cache sized for ``max_new_tokens`` more positions)."""
        self._require("prefill", "colocated")
        B, S = tokens.shape
        kv = KVCache(self.arch, B, S + max_new_tokens, tokens.device)
        return self.executor.forward(tokens, kv=kv), kv

    @torch.no_grad()
    def decode(self, tokens: torch.Tensor, kv: KVCache) -> torch.Tensor:
        """One decode step for the newest token of each sequence -> fp32 logits."""
        self._require("decode", "colocated")
        return self.executor.decode(tokens, kv)

    @torch.no_grad()
    def generate(self, kv: KVCache, first_tokens: torch.Tensor, steps: int) -> tuple[torch.Tensor, list]:
        """Greedy decode ``steps`` tokens after a prefill; returns (tokens [B, steps],
        per-step fp32 logits)."""
        out, logits = [], []
        tok = first_tokens
        for _ in range(steps):
            lg = self.decode(tok, kv)
            logits.append(lg)
            tok = lg.argmax(-1)
            out.append(tok)
        return torch.stack(out, 1), logits

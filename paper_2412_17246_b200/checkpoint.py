"""Checkpoints -> layer slabs: the on-disk path into the O(1) host cache.

The reference has no weight format (a model is ``num_layers x bytes_per_layer``,
parampool.py:25-62) and models the SSD path as a bandwidth (autoscaler.py:113-117).
Here a Hugging Face Llama checkpoint in safetensors (``model.layers.{i}.self_attn.q_proj.weight``
...) is packed into the slab layout of ``slab.py`` -- q/k/v and gate/up fused
row-wise exactly as the GEMMs read them -- directly inside the pinned host
cache, so loading a real checkpoint is one sequential pass over the files and
the copy engines take it from there.

``save_llama`` writes the inverse (used for round-trip tests and to produce
synthetic checkpoints offline).
"""

from __future__ import annotations

import json
import time
from pathlib import Path

import torch

from .llama import SlabWeights
from .slab import LlamaArch, SlabLayout


def _hf_names(arch: LlamaArch, k: int) -> dict[str, list[str]]:
    """Slab tensor -> HF tensor names concatenated along rows (in order)."""
    p = f"model.layers.{k}."
    out = {
        "attn_norm": [p + "input_layernorm.weight"],
        "wqkv": [p + "self_attn.q_proj.weight", p + "self_attn.k_proj.weight",
                 p + "self_attn.v_proj.weight"],
        "wo": [p + "self_attn.o_proj.weight"],
        "ffn_norm": [p + "post_attention_layernorm.weight"],
        "wgu": [p + "mlp.gate_proj.weight", p + "mlp.up_proj.weight"],
        "wdown": [p + "mlp.down_proj.weight"],
    }
    if k == 0:
        out["embed"] = ["model.embed_tokens.weight"]
    if k == arch.n_layers - 1:
        out["final_norm"] = ["model.norm.weight"]
        out["lm_head"] = ["lm_head.weight"]
    return out


def save_llama(weights: SlabWeights, directory, shard_bytes: int = 2 << 30) -> list[Path]:
    """Write the slab's model as HF-named bf16 safetensors shards (+ index)."""
    from safetensors.torch import save_file

    directory = Path(directory)
    directory.mkdir(parents=True, exist_ok=True)
    arch = weights.arch
    tensors: dict[str, torch.Tensor] = {}
    for k, views in enumerate(weights.layers):
        for slab_name, hf in _hf_names(arch, k).items():
            t = views[slab_name].detach().cpu()
            if len(hf) == 1:
                tensors[hf[0]] = t.clone()
                continue
            sizes = ([arch.d_model, arch.kv_dim, arch.kv_dim] if slab_name == "wqkv"
                     else [arch.ffn, arch.ffn])
            for name, part in zip(hf, torch.split(t, sizes, dim=0)):
                tensors[name] = part.clone()
    files, shard, used, index = [], {}, 0, {}

    def flush():
        nonlocal shard, used
        if shard:
            f = directory / f"model-{len(files) + 1:05d}.safetensors"
            save_file(shard, str(f))
            files.append(f)
            for n in shard:
                index[n] = f.name
            shard, used = {}, 0

    for name, t in tensors.items():
        nbytes = t.numel() * t.element_size()
        if used and used + nbytes > shard_bytes:
            flush()
        shard[name] = t
        used += nbytes
    flush()
    (directory / "model.safetensors.index.json").write_text(
        json.dumps({"metadata": {"format": "pt"}, "weight_map": index}, indent=1))
    return files


def load_llama_into(buffer: torch.Tensor, arch: LlamaArch, layout: SlabLayout, directory,
                    tp_rank: int = 0, tp: int = 1) -> dict:
    """Pack an HF safetensors checkpoint into ``buffer`` (uint8, slab layout).

    ``buffer`` is typically ``HostCache.tensor`` (pinned); returns read stats.
    Only TP=1 packing is implemented (a TP shard would slice rows/cols per rank).
    """
    if tp != 1:
        raise NotImplementedError("TP checkpoint sharding is not implemented")
    from safetensors import safe_open

    directory = Path(directory)
    index = json.loads((directory / "model.safetensors.index.json").read_text())["weight_map"]
    view = SlabWeights(arch, layout, buffer)
    handles: dict[str, object] = {}
    t0 = time.perf_counter()
    nbytes = 0
    try:
        for k, views in enumerate(view.layers):
            for slab_name, hf in _hf_names(arch, k).items():
                dst = views[slab_name]
                row = 0
                for name in hf:
                    fname = index[name]
                    if fname not in handles:
                        handles[fname] = safe_open(str(directory / fname), framework="pt")
                    t = handles[fname].get_tensor(name)
                    if t.dtype != torch.bfloat16:
                        t = t.to(torch.bfloat16)
                    rows = t.shape[0] if t.dim() > 1 else t.numel()
                    if dst.dim() == 1:
                        dst.copy_(t)
                    else:
                        dst[row:row + rows].copy_(t)
                    row += rows
                    nbytes += t.numel() * 2
                if dst.dim() > 1 and row != dst.shape[0]:
                    raise ValueError(f"layer {k} {slab_name}: {row} rows packed, expected {dst.shape[0]}")
    finally:
        handles.clear()
    secs = time.perf_counter() - t0
    return {"bytes": nbytes, "seconds": secs, "GBps": nbytes / secs / 1e9 if secs > 0 else None}

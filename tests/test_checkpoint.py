"""HF safetensors checkpoint <-> layer slab packing (CPU round trip)."""

import torch

from paper_2412_17246_b200 import slab as S
from paper_2412_17246_b200.checkpoint import load_llama_into, save_llama
from paper_2412_17246_b200.llama import SlabWeights


def test_safetensors_round_trip_into_slab(tmp_path):
    arch = S.TINY_4L
    lay = S.SlabLayout.for_arch(arch, tile_bytes=64 * 1024)
    src = torch.zeros(lay.data_bytes, dtype=torch.uint8)
    w = SlabWeights(arch, lay, src)
    g = torch.Generator().manual_seed(0)
    for views in w.layers:
        for t in views.values():
            t.copy_(torch.randn(t.shape, generator=g))
    files = save_llama(w, tmp_path, shard_bytes=8 << 20)
    assert len(files) >= 2  # sharded
    dst = torch.zeros_like(src)
    stats = load_llama_into(dst, arch, lay, tmp_path)
    assert torch.equal(dst, src)
    assert stats["bytes"] == arch.total_bytes()


def test_hf_names_fuse_qkv_and_gate_up():
    from safetensors import safe_open
    import tempfile
    arch = S.TINY_4L
    lay = S.SlabLayout.for_arch(arch, tile_bytes=64 * 1024)
    buf = torch.zeros(lay.data_bytes, dtype=torch.uint8)
    w = SlabWeights(arch, lay, buf)
    w.layers[1]["wqkv"][arch.d_model:arch.d_model + 1].fill_(3.0)   # first k_proj row
    with tempfile.TemporaryDirectory() as d:
        save_llama(w, d)
        import json, pathlib
        idx = json.loads((pathlib.Path(d) / "model.safetensors.index.json").read_text())["weight_map"]
        name = "model.layers.1.self_attn.k_proj.weight"
        with safe_open(str(pathlib.Path(d) / idx[name]), framework="pt") as f:
            k = f.get_tensor(name)
        assert k.shape == (arch.kv_dim, arch.d_model) and float(k[0, 0]) == 3.0

"""tcgen05 causal flash attention (prefill) vs a plain PyTorch fp32 reference.

Reference: softmax(q k^T / sqrt(hd) + causal mask) v in fp32 over the same bf16
q / k / v (GQA by repeating kv heads).  Tolerance: the kernel rounds P to bf16
for the P.V product and stores bf16, so relative L2 error <= 1e-2 and max
elementwise error <= 2e-2 of max|ref|.
"""

import ctypes
import math

import pytest
import torch

from paper_2412_17246_b200._native import cuda_lib

pytestmark = pytest.mark.gpu


def flash(qkv, B, S, H, KV, hd):
    lib = cuda_lib()
    need = ctypes.c_int64()
    lib.bz_prefill_attention_workspace_bytes(B, S, KV, hd, ctypes.byref(need))
    ws = torch.full((need.value,), 0xFF, dtype=torch.uint8, device="cuda")   # NaN garbage: the pad must be zeroed
    out = torch.empty(B * S, H * hd, dtype=torch.bfloat16, device="cuda")
    lib.bz_prefill_attention(qkv.data_ptr(), qkv.stride(0), B, S, H, KV, hd, ws.data_ptr(), need.value,
                             out.data_ptr(), out.stride(0), torch.cuda.current_stream().cuda_stream)
    return out


def reference(qkv, B, S, H, KV, hd):
    x = qkv.float().view(B, S, -1)
    q = x[..., :H * hd].view(B, S, H, hd).transpose(1, 2)
    k = x[..., H * hd:(H + KV) * hd].view(B, S, KV, hd).transpose(1, 2)
    v = x[..., (H + KV) * hd:(H + 2 * KV) * hd].view(B, S, KV, hd).transpose(1, 2)
    k = k.repeat_interleave(H // KV, dim=1)
    v = v.repeat_interleave(H // KV, dim=1)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(hd)
    s = s.masked_fill(torch.ones(S, S, dtype=torch.bool, device=s.device).triu(1), float("-inf"))
    return (torch.softmax(s, -1) @ v).transpose(1, 2).reshape(B * S, H * hd)


@pytest.mark.parametrize("B,S,H,KV,hd,extra", [
    (2, 2000, 32, 32, 128, 0),     # Llama-2 7B prefill shape
    (1, 1024, 32, 8, 128, 0),      # GQA 4:1
    (2, 300, 8, 1, 128, 64),       # ragged S (not a tile multiple), MQA, padded row stride
    (3, 64, 4, 4, 64, 0),          # tiny-4l shape (hd 64), S < one tile
    (2, 129, 4, 2, 64, 0),         # one row past a tile boundary
    (1, 1, 2, 2, 128, 0),          # a single token
])
def test_flash_prefill_matches_fp32(B, S, H, KV, hd, extra):
    torch.manual_seed(B * 1000 + S + H)
    width = (H + 2 * KV) * hd
    qkv = (torch.randn(B * S, width + extra, device="cuda") * 1.5).to(torch.bfloat16)[:, :width]
    got = flash(qkv, B, S, H, KV, hd)
    torch.cuda.synchronize()
    want = reference(qkv, B, S, H, KV, hd)
    assert not torch.isnan(got).any()
    err = got.float() - want
    assert (err.norm() / want.norm()).item() <= 1e-2
    assert (err.abs().max() / want.abs().max()).item() <= 2e-2

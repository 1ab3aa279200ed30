"""Prefill attention: tcgen05 flash kernel vs torch SDPA (cuDNN) at Llama-2 7B shapes.
TF/s counts the causal half: 2 * 2 * B * H * S^2 * hd / 2 flop."""
import ctypes, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2412_17246_b200._native import cuda_lib

def run(B, S, H=32, KV=32, hd=128, iters=20):
    lib = cuda_lib(0)
    qkv = torch.randn(B * S, (H + 2 * KV) * hd, device="cuda").to(torch.bfloat16)
    need = ctypes.c_int64()
    lib.bz_prefill_attention_workspace_bytes(B, S, KV, hd, ctypes.byref(need))
    ws = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    out = torch.empty(B * S, H * hd, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ours = lambda: lib.bz_prefill_attention(qkv.data_ptr(), qkv.stride(0), B, S, H, KV, hd, ws.data_ptr(),
                                            need.value, out.data_ptr(), out.stride(0), s)
    x = qkv.view(B, S, -1)
    q = x[..., :H * hd].view(B, S, H, hd).transpose(1, 2)
    k = x[..., H * hd:(H + KV) * hd].view(B, S, KV, hd).transpose(1, 2)
    v = x[..., (H + KV) * hd:].view(B, S, KV, hd).transpose(1, 2)
    att = torch.empty(B * S, H * hd, dtype=torch.bfloat16, device="cuda")
    def sdpa():
        o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=KV != H)
        att.copy_(o.transpose(1, 2).reshape(B * S, H * hd))
    res = {"B": B, "S": S, "H": H, "KV": KV, "hd": hd}
    flop = 2 * 2 * B * H * S * S * hd / 2
    for name, fn in (("tcgen05_flash", ours), ("torch_sdpa_plus_copy", sdpa)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res[name] = {"us": ms * 1e3, "TFLOPs": flop / ms / 1e9}
    torch.cuda.synchronize()
    return res

if __name__ == "__main__":
    for B, S, H, KV in ((1, 2000, 32, 32), (4, 2000, 32, 32), (8, 512, 32, 32), (2, 2048, 64, 8), (12, 2000, 32, 32)):
        print(json.dumps(run(B, S, H, KV)), flush=True)

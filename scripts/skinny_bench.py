"""Decode-shaped GEMMs: ours (stream-K, tcgen05) vs cuBLAS (torch.matmul), GB/s of weights."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200._native import cuda_lib  # noqa: E402

lib = cuda_lib()
ws = torch.zeros((32 << 20) // 4, dtype=torch.float32, device="cuda")
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096), "down": (4096, 11008),
          "lm_head": (32000, 4096)}
ms = [int(x) for x in sys.argv[1:]] or [1, 8, 64]
ctas = ctypes.c_int(0)
for m in ms:
    for name, (n, k) in shapes.items():
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        bs = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(4)]  # > L2 in rotation
        c = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def ours(b):
            lib.bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, m, n, k, k, k, n, 0, 0, 1,
                                ws.data_ptr(), 32 << 20, None, ctypes.byref(ctas), s)

        def cublas(b):
            torch.matmul(a, b.t(), out=c)

        res = {}
        for label, fn in (("ours", ours), ("cublas", cublas)):
            for i in range(8):
                fn(bs[i % 4])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            iters = 40
            for i in range(iters):
                fn(bs[i % 4])
            e1.record()
            e1.synchronize()
            us = e0.elapsed_time(e1) / iters * 1e3
            res[label] = {"us": round(us, 2), "GBps": round(n * k * 2 / us / 1e3, 1)}
        print(json.dumps({"m": m, "shape": name, "ctas": ctas.value, **res}))

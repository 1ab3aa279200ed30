"""Prefill GEMMs at smaller token counts (M = 256 .. 1024) vs cuBLAS: TFLOP/s."""
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200._native import cuda_lib  # noqa: E402


def bench(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / iters


lib = cuda_lib()
st = torch.cuda.current_stream().cuda_stream
WS = 64 << 20  # as LlamaExecutor: enables the skinny/split-K schedules
ws = torch.zeros(WS // 4, dtype=torch.float32, device="cuda")
ctas = ctypes.c_int(0)
MS = [int(x) for x in __import__("os").environ.get("BZ_MS", "256,384,512,768,1024,1536").split(",")]
for m in MS:
    for name, (n, k) in {"qkv": (12288, 4096), "o": (4096, 4096), "gate_up": (22016, 4096),
                         "down": (4096, 11008)}.items():
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ms = bench(lambda: lib.bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, m, n, k, k, k, n,
                                               0, 0, 1, ws.data_ptr(), WS, None, ctypes.byref(ctas), st))
        ref = bench(lambda: torch.matmul(a, b.t()))
        err = float(((c.float() - a.float() @ b.float().t()).abs().max() / (a.float() @ b.float().t()).abs().max()))
        f = 2.0 * m * n * k
        print(json.dumps({"m": m, "shape": name, "ctas": ctas.value, "ours_tf": round(f / ms / 1e9, 1),
                          "cublas_tf": round(f / ref / 1e9, 1), "ratio": round(ref / ms, 3), "err": err}))

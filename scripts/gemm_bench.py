"""Throughput of the tcgen05 GEMM on the Llama-2 7B block shapes (and 8192^3),
next to torch.matmul (cuBLAS) on the same operands.  CUDA-event timed, warm."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200._native import cuda_lib  # noqa: E402

SHAPES = {  # name: (M, N, K)
    "qkv@2000": (2000, 12288, 4096),
    "o@2000": (2000, 4096, 4096),
    "gate_up@2000": (2000, 22016, 4096),
    "down@2000": (2000, 4096, 11008),
    "lm_head@16": (16, 32000, 4096),
    "sq8192": (8192, 8192, 8192),
}


def bench(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / iters


def main():
    lib = cuda_lib()
    out = {}
    for name, (m, n, k) in SHAPES.items():
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        st = torch.cuda.current_stream().cuda_stream

        def ours():
            lib.bz_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, m, n, k, k, k, n, 0, 0, st)

        ms = bench(ours)
        ms_ref = bench(lambda: torch.matmul(a, b.t()))
        flops = 2.0 * m * n * k
        err = ((c.float() - a.float() @ b.float().t()).abs().max() /
               (a.float() @ b.float().t()).abs().max()).item()
        out[name] = {"M": m, "N": n, "K": k, "ms": ms, "tflops": flops / ms / 1e9,
                     "cublas_ms": ms_ref, "cublas_tflops": flops / ms_ref / 1e9, "max_rel_err": err}
        print(json.dumps({name: out[name]}), flush=True)


if __name__ == "__main__":
    main()

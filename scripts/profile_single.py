"""Single-GPU workload for ncu captures of the data-plane movers and the GEMM.

  push      : one chain hop of the Llama-2 7B slab, slab -> slab on this GPU
              (k_push_tiles / k_push_tiles_tma with the relay tracker)
  gemm      : the 7B block GEMMs at 2000 tokens (k_gemm_bf16)
  block     : one full 7B Llama block forward (GEMMs + glue kernels + SDPA)
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2412_17246_b200 as ss  # noqa: E402
from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200._native import cuda_lib  # noqa: E402
from paper_2412_17246_b200.dataplane import ENGINE_TMA, ENGINE_VECTOR, DeviceSlab, execute_plan_loopback  # noqa: E402


def push(engine):
    lay = S.SlabLayout.for_arch(S.LLAMA2_7B, tile_bytes=1 << 20)
    a, b = DeviceSlab(lay, 0), DeviceSlab(lay, 0)
    a.fill_random(1)
    plan = ss.ScalePlan(edges=[ss.planner.PlanEdge("gpu0", "gpu1", 7200.0, "nvlink")],
                        chains=[["gpu0", "gpu1"]])
    for e in range(1, 5):
        execute_plan_loopback(plan, {"gpu0": a, "gpu1": b}, e, engine=engine, nctas=32)
    torch.cuda.synchronize()
    assert torch.equal(a.fingerprints(), b.fingerprints())
    a.close()
    b.close()


def gemm():
    lib = cuda_lib()
    st = torch.cuda.current_stream().cuda_stream
    for (m, n, k) in [(2000, 12288, 4096), (2000, 22016, 4096), (2000, 4096, 11008)]:
        x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        w = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
        c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        for _ in range(3):
            lib.bz_gemm_bf16(x.data_ptr(), w.data_ptr(), c.data_ptr(), None, m, n, k, k, k, n, 0, 0, st)
    torch.cuda.synchronize()


def block():
    from paper_2412_17246_b200.llama import LlamaExecutor, SlabWeights
    arch = S.LlamaArch("llama2-7b-2l", 4096, 2, 32, 32, 11008)
    lay = S.SlabLayout.for_arch(arch, tile_bytes=1 << 20)
    s = DeviceSlab(lay, 0)
    w = SlabWeights(arch, lay, s.data)
    w.init_random(0)
    ex = LlamaExecutor(w, max_tokens=2000, device="cuda")
    toks = torch.randint(0, arch.vocab, (4, 500), device="cuda")
    for _ in range(3):
        ex.forward(toks)
    torch.cuda.synchronize()
    s.close()


if __name__ == "__main__":
    what = sys.argv[1:] or ["push", "gemm", "block"]
    for w in what:
        if w == "push":
            push(ENGINE_VECTOR)
        elif w == "push_tma":
            push(ENGINE_TMA)
        elif w == "gemm":
            gemm()
        elif w == "block":
            block()
    print("ok", what)

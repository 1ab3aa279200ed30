"""tcgen05/TMEM/TMA GEMM numerics vs a plain PyTorch fp32 reference.

C = A . B^T with bf16 inputs, fp32 accumulation: compared with the fp32 matmul
of the same bf16 values; tolerance = bf16 output rounding (rel 1e-2 on the
max-normalised error) -- the north star's cooperative-logit tolerance.
"""

import pytest
import torch

from paper_2412_17246_b200._native import BZ_GEMM_B_STATIC, BZ_GEMM_C_F32, cuda_lib

pytestmark = pytest.mark.gpu


def gemm(a, b, residual=None, max_ctas=0):
    m, k = a.shape
    n = b.shape[0]
    c = torch.empty(m, n, dtype=torch.bfloat16, device=a.device)
    cuda_lib().bz_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(),
                            residual.data_ptr() if residual is not None else None,
                            m, n, k, a.stride(0), b.stride(0), c.stride(0),
                            residual.stride(0) if residual is not None else 0, max_ctas,
                            torch.cuda.current_stream().cuda_stream)
    return c


def _check(c, ref):
    err = (c.float() - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err / scale < 1e-2, (err, scale)


@pytest.mark.parametrize("m,n,k", [
    (128, 256, 64), (128, 256, 128), (256, 512, 512), (2000, 4096, 4096), (7, 24, 64),
    (300, 1000, 192), (2000, 12288, 4096), (2000, 4096, 11008), (33, 32000, 256),
    (64, 256, 688), (200, 1376, 256), (129, 264, 40),
])
def test_gemm_matches_fp32(m, n, k):
    torch.manual_seed(m * 7 + n + k)
    a = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    c = gemm(a, b)
    torch.cuda.synchronize()
    _check(c, a.float() @ b.float().t())


def test_gemm_residual_epilogue():
    torch.manual_seed(1)
    a = torch.randn(512, 1024, device="cuda").to(torch.bfloat16)
    b = (torch.randn(768, 1024, device="cuda") * 0.03).to(torch.bfloat16)
    r = torch.randn(512, 768, device="cuda").to(torch.bfloat16)
    c = gemm(a, b, residual=r)
    torch.cuda.synchronize()
    _check(c, a.float() @ b.float().t() + r.float())


def test_gemm_strided_operands_and_few_ctas():
    torch.manual_seed(2)
    big = torch.randn(256, 640, device="cuda").to(torch.bfloat16)
    a = big[:, 64:576]                      # lda = 640
    b = (torch.randn(384, 512, device="cuda") * 0.05).to(torch.bfloat16)
    c = gemm(a, b, max_ctas=3)
    torch.cuda.synchronize()
    _check(c, a.float() @ b.float().t())


def test_gemm_exact_small_integers():
    """Integer-valued operands: fp32 accumulation must be exact."""
    a = torch.randint(-3, 4, (256, 640), device="cuda").to(torch.bfloat16)
    b = torch.randint(-3, 4, (512, 640), device="cuda").to(torch.bfloat16)
    c = gemm(a, b)
    torch.cuda.synchronize()
    assert torch.equal(c, (a.float() @ b.float().t()).to(torch.bfloat16))


def gemm_ex(a, b, residual=None, ws_bytes=32 << 20, signal=None):
    import ctypes
    m, k = a.shape
    n = b.shape[0]
    c = torch.empty(m, n, dtype=torch.bfloat16, device=a.device)
    ws = torch.zeros(max(ws_bytes, 16) // 4, dtype=torch.float32, device=a.device)
    ctas = ctypes.c_int(0)
    cuda_lib().bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(),
                               residual.data_ptr() if residual is not None else None,
                               m, n, k, a.stride(0), b.stride(0), c.stride(0),
                               residual.stride(0) if residual is not None else 0, 0, 1,
                               ws.data_ptr() if ws_bytes else None, ws_bytes,
                               signal.data_ptr() if signal is not None else None, ctypes.byref(ctas),
                               torch.cuda.current_stream().cuda_stream)
    return c, ctas.value


@pytest.mark.parametrize("m,n,k", [
    (1, 4096, 4096), (1, 12288, 4096), (8, 4096, 11008), (64, 22016, 4096), (1, 32000, 4096),
    (16, 256, 688), (3, 264, 4104), (128, 4096, 4096), (32, 4096, 4096), (64, 4096, 11008),
    (2, 96, 4096), (5, 40, 64), (1, 1376, 256), (4, 22016, 4096), (16, 15360, 5120),
])
def test_streamk_skinny_gemm_matches_fp32(m, n, k):
    """Decode-shaped GEMMs (M = batch rows) run stream-K: tiles shared by CTAs are summed in fp32."""
    torch.manual_seed(m + n + k)
    a = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    r = torch.randn(m, n, device="cuda").to(torch.bfloat16)
    ref = a.float() @ b.float().t()
    c, _ = gemm_ex(a, b)
    c2, _ = gemm_ex(a, b, residual=r)
    c0, _ = gemm_ex(a, b, ws_bytes=0)           # no workspace: no split
    torch.cuda.synchronize()
    _check(c, ref)
    _check(c2, ref + r.float())
    _check(c0, ref)


def test_streamk_workspace_left_zeroed_and_reusable():
    """Tile arrival counters are reset by the last slice: the same workspace
    serves back-to-back calls (as in a replayed decode graph)."""
    import ctypes
    torch.manual_seed(6)
    a = (torch.randn(4, 4096, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    ws = torch.zeros((8 << 20) // 4, dtype=torch.float32, device="cuda")
    c = torch.empty(4, 4096, dtype=torch.bfloat16, device="cuda")
    ctas = ctypes.c_int(0)
    for _ in range(3):
        cuda_lib().bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, 4, 4096, 4096, 4096, 4096,
                                   4096, 0, 0, 0, ws.data_ptr(), 8 << 20, None, ctypes.byref(ctas),
                                   torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        _check(c, a.float() @ b.float().t())
    assert int(ws[:64].view(torch.int32).abs().sum().item()) == 0


def test_streamk_signal_counts_every_cta():
    torch.manual_seed(5)
    a = (torch.randn(2, 4096, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    sig = torch.zeros(1, dtype=torch.int32, device="cuda")
    c, ctas = gemm_ex(a, b, signal=sig)
    torch.cuda.synchronize()
    assert ctas > 0 and int(sig.item()) == ctas
    _check(c, a.float() @ b.float().t())


@pytest.mark.parametrize("m,n,k", [(256, 4096, 4096), (300, 4096, 11008), (512, 4096, 4096), (384, 1024, 8192)])
def test_pair_splitk_prefill_shapes(m, n, k):
    """Short-prompt prefill GEMMs (few 256-row pair tiles, long K) split K into fp32
    partials reduced by a second pass, with the residual and the hand-off signal."""
    torch.manual_seed(m + n + k)
    a = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    r = torch.randn(m, n, device="cuda").to(torch.bfloat16)
    sig = torch.zeros(1, dtype=torch.int32, device="cuda")
    c, ctas = gemm_ex(a, b, residual=r, ws_bytes=64 << 20, signal=sig)
    torch.cuda.synchronize()
    _check(c, a.float() @ b.float().t() + r.float())
    assert ctas > 0 and int(sig.item()) == ctas


@pytest.mark.parametrize("m,n,k,ws", [(4, 32000, 4096, True), (8, 32000, 4096, False), (200, 4096, 512, False),
                                      (1, 1000, 256, True)])
def test_gemm_fp32_output(m, n, k, ws):
    """BZ_GEMM_C_F32 (logit heads): the accumulator is stored unrounded -- far tighter
    than the bf16 rounding bound (fp32 accumulation order is the only difference),
    whole-tile and stream-K (workspace) schedules alike."""
    from paper_2412_17246_b200._native import BZ_GEMM_B_STATIC, BZ_GEMM_C_F32
    import ctypes
    torch.manual_seed(m + n)
    a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    c = torch.full((m, n), float("nan"), dtype=torch.float32, device="cuda")
    w = torch.zeros(16 << 20, dtype=torch.float32, device="cuda") if ws else None
    cuda_lib().bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, m, n, k, a.stride(0), b.stride(0),
                               c.stride(0), 0, 0, BZ_GEMM_B_STATIC | BZ_GEMM_C_F32,
                               w.data_ptr() if w is not None else None, (w.numel() * 4) if w is not None else 0,
                               None, ctypes.byref(ctypes.c_int()), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    assert not torch.isnan(c).any()
    assert ((c - ref).abs().max() / ref.abs().max()).item() < 1e-4


def test_splitk_partials_leave_streamk_counters_zero():
    """Regression: the pair kernel's split-K partials and the stream-K tile counters
    share one workspace.  A split-K prefill GEMM (down projection, 256 tokens) followed
    by a stream-K decode GEMM (4 rows) on the same workspace must both be exact, and
    the counter header must read zero afterwards (it used to be overwritten by fp32
    partials, so the next decode step summed garbage)."""
    from paper_2412_17246_b200._native import BZ_GEMM_B_STATIC
    import ctypes
    torch.manual_seed(5)
    ws = torch.zeros(64 << 20 >> 2, dtype=torch.float32, device="cuda")

    def run(a, b):
        c = torch.empty(a.shape[0], b.shape[0], dtype=torch.bfloat16, device="cuda")
        cuda_lib().bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(), None, a.shape[0], b.shape[0],
                                   a.shape[1], a.stride(0), b.stride(0), c.stride(0), 0, 0, BZ_GEMM_B_STATIC,
                                   ws.data_ptr(), ws.numel() * 4, None, ctypes.byref(ctypes.c_int()),
                                   torch.cuda.current_stream().cuda_stream)
        return c

    for _ in range(2):
        a1 = torch.randn(256, 11008, device="cuda").to(torch.bfloat16)
        b1 = (torch.randn(4096, 11008, device="cuda") * 0.02).to(torch.bfloat16)
        c1 = run(a1, b1)
        a2 = torch.randn(4, 4096, device="cuda").to(torch.bfloat16)
        b2 = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
        c2 = run(a2, b2)
        torch.cuda.synchronize()
        _check(c1, a1.float() @ b1.float().t())
        _check(c2, a2.float() @ b2.float().t())
        assert int(ws[:1024].view(torch.int32).abs().sum()) == 0


def _gemm_flags(a, b, residual=None, c_f32=False, signal=None, max_ctas=0):
    import ctypes
    m, k = a.shape
    n = b.shape[0]
    c = torch.empty(m, n, dtype=torch.float32 if c_f32 else torch.bfloat16, device=a.device)
    ctas = ctypes.c_int(0)
    cuda_lib().bz_gemm_bf16_ex(a.data_ptr(), b.data_ptr(), c.data_ptr(),
                               residual.data_ptr() if residual is not None else None,
                               m, n, k, a.stride(0), b.stride(0), c.stride(0),
                               residual.stride(0) if residual is not None else 0, max_ctas,
                               BZ_GEMM_B_STATIC | (BZ_GEMM_C_F32 if c_f32 else 0), None, 0,
                               signal.data_ptr() if signal is not None else None, ctypes.byref(ctas),
                               torch.cuda.current_stream().cuda_stream)
    return c, ctas.value


@pytest.mark.parametrize("split", [1, 2, 3, 4, 5, 6, 7, 8])
def test_swapped_decode_gemm_every_cluster_split(monkeypatch, split):
    """Decode GEMMs (M <= 16) with the weight tile as the MMA's M operand and K split
    over a cluster of `split` CTAs (partials summed in distributed shared memory):
    ragged N (not a multiple of 128), an odd number of 2-k-block chunks, residual,
    fp32 C and the per-CTA completion signal; the fixed summation order makes a
    repeated call bit-identical."""
    monkeypatch.setenv("BZ_GEMM_SWAP_S", str(split))
    torch.manual_seed(split)
    m, n, k = 13, 1000, 64 * 37
    a = (torch.randn(m, k, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(n, k, device="cuda") * 0.02).to(torch.bfloat16)
    r = torch.randn(m, n, device="cuda").to(torch.bfloat16)
    ref = a.float() @ b.float().t()
    sig = torch.zeros(1, dtype=torch.int32, device="cuda")
    c, ctas = _gemm_flags(a, b, residual=r, signal=sig)
    c_again, _ = _gemm_flags(a, b, residual=r)
    f, _ = _gemm_flags(a, b, c_f32=True)
    torch.cuda.synchronize()
    assert ctas == 8 * split and int(sig.item()) == ctas
    _check(c, ref + r.float())
    assert torch.equal(c, c_again)
    assert (f - ref).abs().max().item() <= 1e-3 * ref.abs().max().item()


@pytest.mark.parametrize("m", [1, 2, 8, 16])
def test_swapped_decode_gemm_respects_cta_cap(m):
    """The split is chosen so tiles x split stays within max_ctas (the co-operative
    decode leaves SMs to the data plane)."""
    torch.manual_seed(m)
    a = (torch.randn(m, 4096, device="cuda") * 0.5).to(torch.bfloat16)
    b = (torch.randn(4096, 4096, device="cuda") * 0.02).to(torch.bfloat16)
    for cap in (0, 100, 40, 32):
        c, ctas = _gemm_flags(a, b, max_ctas=cap)
        torch.cuda.synchronize()
        assert 0 < ctas <= (cap or 148)
        _check(c, a.float() @ b.float().t())

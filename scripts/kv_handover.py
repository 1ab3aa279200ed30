"""KV hand-over bandwidth: a 7B cooperative pair's source-side KV blocks
(16 of 32 layers, 4 sequences x 2048 cached tokens) copied cuda:0 -> cuda:1 with
bz_copy_panels (peer stores over NVLink), vs the same bytes with torch's peer copy."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200._native import cuda_lib  # noqa: E402

lib = cuda_lib()
lib.bz_enable_peer_mesh(0)
lib.bz_enable_peer_mesh(1)
B, KV, S_MAX, LEN, HD, LAYERS = 4, 32, 2304, 2048, 128, 16
src = [torch.randn(B, KV, S_MAX, HD, device="cuda:0").to(torch.bfloat16) for _ in range(2 * LAYERS)]
dst = [torch.empty(B, KV, S_MAX, HD, device="cuda:1", dtype=torch.bfloat16) for _ in range(2 * LAYERS)]
stride, prefix = S_MAX * HD * 2, LEN * HD * 2
nbytes = 2 * LAYERS * B * KV * prefix
out = {"bytes": nbytes}
for nctas in (32, 64, 128):
    with torch.cuda.device(0):
        s = torch.cuda.current_stream()
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for a, b in zip(src, dst):
                lib.bz_copy_panels(a.data_ptr(), b.data_ptr(), B * KV, stride, stride, prefix, nctas, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
        out[f"copy_panels_{nctas}ctas_GBps"] = nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
ok = all(torch.equal(a[:, :, :LEN].cpu(), b[:, :, :LEN].cpu()) for a, b in zip(src[:2], dst[:2]))
with torch.cuda.device(0):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for a, b in zip(src, dst):
        b[:, :, :LEN].copy_(a[:, :, :LEN])
    e1.record()
    e1.synchronize()
out["torch_peer_copy_GBps"] = nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
out["bit_exact"] = ok
print(json.dumps(out))

"""Measured pair-throughput ramp vs the reference's steady_state_throughput (2 GPUs).

  python scripts/ramp.py [arch] [batches]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.ramp import measure_ramp  # noqa: E402

arch = S.ARCHS[sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 16
r = measure_ramp(arch, batches=n)
for p in r["points"]:
    print(f"k={p['k']:3d}  measured {p['measured_rel']:.3f}  reference {p['reference_rel']:.3f}  "
          f"({p['measured_batches_per_s']:.2f} batches/s)", flush=True)
print(json.dumps(r))

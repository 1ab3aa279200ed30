"""Interference between serving (KV-cache) traffic and scale traffic on NVLink, and
what the planner's source pruning buys (planner.py:147-159,
265-285).  Run under torchrun with 4 GPUs:

  gpu0 = prefill instance, continuously pushing KV cache to gpu1 (decode);
  gpu1 = decode instance; both hold the Llama-2 7B weights;
  gpu2, gpu3 = new instances to scale up.

Case "pruned": the FlowSet carries the kvcache flow gpu0->gpu1 at its measured
rate (paper_2412_17246_b200/interference.py, kvflows.MeasuredFlow), so
generate_plan(prune=True) drops gpu0 and scales from gpu1 (its NVLink egress
is idle -- only its ingress carries KV).  Case "naive": the plan is forced to
use gpu0, whose egress is shared with the KV stream.  Reported: scale-up time,
and the KV stream's throughput while the scale-up runs vs alone.
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2412_17246_b200.dataplane import Fabric  # noqa: E402

def main():
    from paper_2412_17246_b200.interference import run_interference
    fabric = Fabric.from_env()
    out = run_interference(fabric)
    if fabric.rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "300")), exit=True)
    main()

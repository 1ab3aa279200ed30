"""Run the two-process live pair (ZigZag while the new instance loads) under torchrun.

  BZ_ARCH=llama2-7b BZ_MODE=host|nvlink BZ_BATCHES=12 python -m torch.distributed.run \
      --nproc-per-node 2 scripts/live_pair.py
Prints one JSON line (rank 0) with executed / predicted average latencies.
"""

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2412_17246_b200 import slab as S  # noqa: E402
from paper_2412_17246_b200.dataplane import Fabric  # noqa: E402
from paper_2412_17246_b200.livepair import LivePair, summarize  # noqa: E402


def main():
    fabric = Fabric.from_env()
    arch = S.ARCHS[os.environ.get("BZ_ARCH", "llama2-7b")]
    pair = LivePair(fabric, arch, n_batches=int(os.environ.get("BZ_BATCHES", "12")),
                    seqs=int(os.environ.get("BZ_SEQS", "4")), seq_len=int(os.environ.get("BZ_SEQ", "500")),
                    mode=os.environ.get("BZ_MODE", "host"), nctas=int(os.environ.get("BZ_NCTAS", "48")),
                    engine={"vector": 0, "vec256": 2, "ce": 3}[os.environ.get("BZ_ENGINE", "vector")])
    res = pair.run()
    ho = pair.run_handover(pair.cfg, pair.tl)
    if res is not None:
        print(json.dumps({"arch": arch.name, **summarize(res), "kv_handover": ho}), flush=True)
    pair.close()
    import torch.distributed as dist
    dist.destroy_process_group()


if __name__ == "__main__":
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("BZ_WATCHDOG_S", "300")), exit=True)
    main()

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

LIB_DIR = ROOT / "paper_2412_17246_b200" / "_lib"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a)")
    config.addinivalue_line("markers", "multigpu: needs >= 2 GPUs")
    # the host decision library is tiny (g++, ~1 s); build it if a fresh checkout lacks it
    if not (LIB_DIR / "libblitz_host.so").exists():
        subprocess.run(["make", "-C", str(ROOT / "paper_2412_17246_b200" / "csrc"), "host"],
                       check=True, capture_output=True)


def cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)

"""ctypes bindings for the two in-tree native libraries.

* ``_lib/libblitz_host.so`` -- CPU decision kernels (``include/blitz_plan.h``).
* ``_lib/libblitz.so``      -- the sm_100a data plane (``include/blitz.h``).

Both are built in-tree by ``make -C paper_2412_17246_b200/csrc`` (called from
``__graft_entry__.build()``).  There is no fallback: if a library is missing,
the call that needs it raises ``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
import math
import os
from pathlib import Path
from typing import Optional, Sequence

LIB_DIR = Path(__file__).resolve().parent / "_lib"
HOST_LIB = LIB_DIR / "libblitz_host.so"
CUDA_LIB = LIB_DIR / "libblitz.so"


class NativeLibraryMissing(RuntimeError):
    pass


def _load(path: Path) -> ctypes.CDLL:
    if not path.exists():
        raise NativeLibraryMissing(
            f"{path.name} is not built; run `make -C {path.parent.parent / 'csrc'}` "
            "or __graft_entry__.build()")
    return ctypes.CDLL(str(path), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)


class _HostLib:
    """Wrapper over libblitz_host.so (include/blitz_plan.h)."""

    def __init__(self):
        self.lib = _load(HOST_LIB)
        f = self.lib.bz_pipeline_dp
        f.restype = ctypes.c_int
        f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                      ctypes.POINTER(ctypes.c_double), ctypes.c_int, ctypes.c_int,
                      ctypes.c_double, ctypes.POINTER(ctypes.c_int)]

    def pipeline_dp(self, batches: int, layers: int, time_l: float, weights: Sequence[float],
                    offset: int, source_prefix: bool, deadline_s: Optional[float]):
        w = (ctypes.c_double * batches)(*weights)
        out = (ctypes.c_int * batches)()
        dl = -1.0 if deadline_s is None else float(deadline_s)
        if dl < 0 and deadline_s is not None:
            dl = 0.0
        rc = self.lib.bz_pipeline_dp(batches, layers, float(time_l), w, int(offset),
                                     1 if source_prefix else 0, dl, out)
        if rc == 0:
            return list(out)
        if rc == 1:
            return None
        if rc == 2:
            return "deadline"
        raise ValueError(f"bz_pipeline_dp rejected its arguments (rc={rc})")


_host: Optional[_HostLib] = None


def host_lib() -> _HostLib:
    global _host
    if _host is None:
        _host = _HostLib()
    return _host

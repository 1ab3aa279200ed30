"""ctypes bindings for the two in-tree native libraries.

* ``_lib/libblitz_host.so`` -- CPU decision kernels (``include/blitz_plan.h``).
* ``_lib/libblitz.so``      -- the sm_100a data plane (``include/blitz.h``).

Both are built in-tree by ``make -C paper_2412_17246_b200/csrc`` (called from
``__graft_entry__.build()``).  There is no fallback: if a library is missing,
the call that needs it raises ``NativeLibraryMissing``.
"""

from __future__ import annotations

import ctypes
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


# ---- libblitz.so (include/blitz.h) ----------------------------------------------------

class BlitzError(RuntimeError):
    """A libblitz call failed; carries bz_last_error()."""


class BzDecodeBlock(ctypes.Structure):
    """bz_decode_block: one block's weight views and KV panels (device pointers)."""
    _fields_ = [(n, ctypes.c_void_p) for n in ("attn_norm", "wqkv", "wo", "ffn_norm", "wgu", "wdown", "k_cache",
                                               "v_cache")]


class BzSlab(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_uint64), ("bytes", ctypes.c_uint64), ("handle", ctypes.c_uint64),
                ("dev", ctypes.c_int), ("fd", ctypes.c_int)]


class BzMc(ctypes.Structure):
    _fields_ = [("handle", ctypes.c_uint64), ("mc_ptr", ctypes.c_uint64), ("bytes", ctypes.c_uint64),
                ("fd", ctypes.c_int)]


_P = ctypes.c_void_p
_I = ctypes.c_int
_U32 = ctypes.c_uint32
_U64 = ctypes.c_uint64
_PP = ctypes.POINTER(ctypes.c_void_p)
_PI = ctypes.POINTER(ctypes.c_int)
_PU64 = ctypes.POINTER(ctypes.c_uint64)

BZ_GEMM_B_STATIC = 1   # include/blitz.h
BZ_GEMM_C_F32 = 2

# name -> argtypes; every function returns int status
_SIGNATURES = {
    "bz_version": [],
    "bz_device_count": [_PI],
    "bz_device_caps": [_I, _PI, _PI, _PI, _PI],
    "bz_enable_peer_mesh": [_I],
    "bz_slab_create": [_I, _U64, ctypes.POINTER(BzSlab)],
    "bz_slab_export": [ctypes.POINTER(BzSlab)],
    "bz_slab_import": [_I, _I, _I, _U64, ctypes.POINTER(BzSlab)],
    "bz_slab_free": [ctypes.POINTER(BzSlab)],
    "bz_mc_granularity": [_I, _I, _PU64, _PU64],
    "bz_mc_create": [_I, _U64, ctypes.POINTER(BzMc)],
    "bz_mc_import": [_I, _I, _U64, ctypes.POINTER(BzMc)],
    "bz_mc_add_device": [ctypes.POINTER(BzMc), _I],
    "bz_mc_bind": [ctypes.POINTER(BzMc), _I, ctypes.POINTER(BzSlab), _U64, _U64, _U64],
    "bz_mc_map": [ctypes.POINTER(BzMc), _I],
    "bz_mc_free": [ctypes.POINTER(BzMc), _I, _U64],
    "bz_mc_unbind": [ctypes.POINTER(BzMc), _I, _U64],
    "bz_pull_tiles": [_P, _P, _P, _P, _P, _P, _I, _I, ctypes.c_uint32, _I, _P],
    "bz_push_tiles_ce_gated": [_P, _P, _P, _P, _P, _I, _I, _I, ctypes.c_uint32, _P, _P, _P],
    "bz_push_tiles": [_P, _PP, _PP, _I, _P, _P, _I, _I, _U32, _I, _I, _P],
    "bz_push_tile_list": [_P, _PP, _PP, _I, _P, _P, _P, _I, _U32, _I, _P],
    "bz_multicast_tiles": [_P, _P, _P, _P, _P, _I, _I, _U32, _I, _P],
    "bz_push_tiles_ce": [_P, _P, _P, _P, _P, _I, _I, _I, _U32, _P],
    "bz_push_tiles_ce2": [_P, _P, _P, _P, _P, _I, _I, _I, _U32, _P, _P],
    "bz_stage_tiles_ce": [_P, _P, _P, _P, _I, _I, _I, _U32, _P],
    "bz_stage_tiles_sm": [_P, _P, _P, _P, _I, _I, _U32, _I, _P],
    "bz_track_layers": [_P, _P, _I, _U32, _P, _P, _P],
    "bz_publish_layer": [_P, _U32, _P, _P],
    "bz_wait_layer": [_P, _U32, _P],
    "bz_wait_flag_kernel": [_P, _U32, _P],
    "bz_wait_timeouts": [_PU64, _U64],
    "bz_fill_random": [_P, _U64, _U64, _P],
    "bz_tile_fingerprints": [_P, _P, _I, _I, _P, _P],
    "bz_handoff": [_P, _P, _U64, _P, _U32, _I, _P],
    "bz_copy_panels": [_P, _P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _I, _P],
    "bz_gemm_bf16": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P],
    "bz_gemm_bf16_signal": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _PI, _P],
    "bz_gemm_bf16_ex": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, ctypes.c_uint, _P, ctypes.c_int64, _P,
                        _PI, _P],
    "bz_rmsnorm": [_P, _P, _P, _I, _I, _I, _I, ctypes.c_float, _P],
    "bz_rope": [_P, _P, _I, _I, _I, _I, ctypes.c_float, _P],
    "bz_silu_mul": [_P, _P, _I, _I, _I, _I, _P],
    "bz_rope_append": [_P, _I, _I, _I, _I, _I, ctypes.c_float, _P, _P, ctypes.c_int64, _P, _P],
    "bz_rope_append_rows": [_P, _I, _I, _I, _I, _I, ctypes.c_float, _P, _P, ctypes.c_int64, _P, _P],
    "bz_decode_workspace_bytes": [_I, _I, _I, _I, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)],
    "bz_decode_attention": [_P, _I, _P, _P, _I, _I, _I, _I, ctypes.c_int64, _P, _P, _I, _P, ctypes.c_int64,
                            _P],
    "bz_decode_attention_rows": [_P, _I, _P, _P, _I, _I, _I, _I, ctypes.c_int64, _P, _P, _I, _P, ctypes.c_int64,
                                 _P],
    "bz_prefill_attention_workspace_bytes": [_I, _I, _I, _I, ctypes.POINTER(ctypes.c_int64)],
    "bz_prefill_attention": [_P, _I, _I, _I, _I, _I, _I, _P, ctypes.c_int64, _P, _I, _P],
    "bz_decode_fused_workspace_bytes": [_I, _I, _I, _I, _I, _I, ctypes.POINTER(ctypes.c_int64)],
    "bz_decode_fused": [ctypes.POINTER(BzDecodeBlock), _I, _P, _I, _I, _I, _I, _I, _I, _I, ctypes.c_float,
                        ctypes.c_float, ctypes.c_int64, _P, _I, _P, ctypes.c_int64, _I, _P],
    "bz_decode_fused_status": [_P, _PI, _P],
    "bz_decode_fused_set_trace": [_P, ctypes.c_int64],
    "bz_sm_count": [_I, _PI],
    "bz_preload_kernels": [_I, _PI],
}


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES) + ["bz_last_error"]


class _CudaLib:
    """Checked wrapper over libblitz.so: every non-zero status raises BlitzError."""

    def __init__(self):
        self.lib = _load(CUDA_LIB)
        self.lib.bz_last_error.restype = ctypes.c_char_p
        self.lib.bz_last_error.argtypes = []
        for name, args in _SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.restype = ctypes.c_int
            fn.argtypes = args

    def __getattr__(self, name):
        if not name.startswith("bz_"):
            raise AttributeError(name)
        fn = getattr(self.lib, name)

        def call(*args):
            rc = fn(*args)
            if rc != 0:
                msg = self.lib.bz_last_error().decode(errors="replace")
                raise BlitzError(f"{name} failed (rc={rc}): {msg}")
            return rc

        call.__name__ = name
        return call


_cuda: Optional[_CudaLib] = None
_preloaded: set = set()


def cuda_lib(device: Optional[int] = None) -> _CudaLib:
    """libblitz.so; raises NativeLibraryMissing if it was not built (no fallback).

    The first call for a device (``device``, else torch's current device once CUDA
    is initialised) loads every libblitz kernel into it (bz_preload_kernels):
    producer and consumer kernels of the data plane run concurrently, and a lazy
    module load at a first launch could otherwise wait on a spinning consumer.
    """
    global _cuda
    if _cuda is None:
        _cuda = _CudaLib()
    if device is None:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            device = torch.cuda.current_device()
    if device is not None and int(device) not in _preloaded:
        n = ctypes.c_int()
        _cuda.bz_preload_kernels(int(device), ctypes.byref(n))
        _preloaded.add(int(device))
    return _cuda


def ptr_array(values: Sequence[int]):
    arr = (ctypes.c_void_p * max(1, len(values)))()
    for i, v in enumerate(values):
        arr[i] = int(v)
    return arr

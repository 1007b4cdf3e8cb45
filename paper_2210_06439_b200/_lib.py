"""ctypes binding of the C ABI in include/sg.h (libsg.so, built in-tree).

There is no CPU fallback: if the library or a CUDA device is missing every
compute entry point raises ``SGUnavailable``.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsg.so"
ABI_VERSION = 4

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_d = ctypes.c_double

# name -> argtypes (restype int unless noted); mirrors include/sg.h
SIGNATURES = {
    "sg_abi_version": [],
    "sg_device_sm_count": [],
    "sg_launch_count": [],
    "sg_cluster_aggregate": [_p, _i64, _i64, _i64, _i64, _d, _p, _p],
    "sg_p2p": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _d, _d, _d, _i32,
               _p, _i64, _i64, _i64, _i64, _i32, _p],
    "sg_m2l": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _p, _i64, _d, _d, _d, _i32, _i32, _i32,
               _p, _i64, _i64, _i64, _i64, _p, _i64, _i32, _p],
    "sg_m2l_workspace_bytes": [_i64],
    "sg_reconstruct": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _d, _p, _p],
    "sg_flux": [_p, _i64, _d, _p, _p, _p, _p, _p, _p, _p, _i32, _p],
    "sg_flux_legacy": [_p, _i64, _d, _p, _p, _p, _p, _p, _p, _p, _i32, _p],
    "sg_hydro_fused": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _d, _d, _p, _p, _p, _p, _p, _p, _p, _i32,
                       _p],
    "sg_hydro_update": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _p, _p, _p, _p, _p, _d, _d, _d,
                        _p, _p, _p, _i32, _p, _p],
    "sg_max_wavespeed": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _d, _d, _p, _p],
    "sg_max_reduce": [_p, _i64, _p, _p],
    "sg_dt_from_smax": [_p, _d, _d, _p, _p],
    "sg_fill_periodic": [_p, _i64, _i64, _i64, _i64, _i32, _i32, _p],
    "sg_gather_blocks": [_p, _i64, _i64, _i64, _i32, _i64, _p, _i64, _i64, _i32, _p, _p],
    "sg_scale_copy": [_p, _i32, _p, _i32, _i64, _i64, _i64, _d, _p],
    "sg_fp64_peak": [ctypes.c_int, ctypes.c_int, _p, ctypes.POINTER(_i64), _p],
    "sg_dropin_max_wavespeed": [_p, _d, _d, _p, _p],
    "sg_dropin_monopole": [_p, _i32, _d, _d, _d, _i32, _p, _p],
    "sg_dropin_multipole": [_p, _d, _d, _d, _i32, _i32, _i32, _i32, _p, _p],
    "sg_dropin_reconstruct": [_p, _d, _p, _p],
    "sg_dropin_flux": [_p, _d, _p, _p, _p, _p, _p, _p],
    "sg_dropin_hydro_update": [_p, _p, _p, _p, _d, _d, _d, _p, _p],
}


RESTYPES = {"sg_m2l_workspace_bytes": _i64, "sg_launch_count": ctypes.c_ulonglong}


class SGUnavailable(RuntimeError):
    """libsg.so or the CUDA device it needs is not available (no fallback)."""


class SGError(RuntimeError):
    """A C-ABI call returned an error code."""


_lib = None

PREC_EXACT, PREC_FMA = 0, 1
PRECISIONS = {"exact": PREC_EXACT, "fma": PREC_FMA}


def load(path: Path | None = None):
    """Load libsg.so (no device needed) and bind every exported symbol."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise SGUnavailable(f"{p} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(str(p))
    for name, argtypes in SIGNATURES.items():
        fn = getattr(L, name)
        fn.argtypes = argtypes
        fn.restype = RESTYPES.get(name, ctypes.c_int)
    L.sg_last_error.argtypes = []
    L.sg_last_error.restype = ctypes.c_char_p
    if L.sg_abi_version() != ABI_VERSION:
        raise SGUnavailable(f"libsg ABI {L.sg_abi_version()} != expected {ABI_VERSION}")
    if path is None:
        _lib = L
    return L


LAUNCHES = {"count": 0}  # ABI calls made through call()


def launch_count() -> int:
    """Kernels actually launched by libsg.so (an ABI call may launch several)."""
    return int(load().sg_launch_count())


def call(name: str, *args) -> None:
    """Invoke an sg_* entry point (each launches exactly one kernel) and raise
    SGError on a non-zero status."""
    L = load()
    LAUNCHES["count"] += 1
    rc = getattr(L, name)(*args)
    if rc != 0:
        raise SGError(f"{name} failed ({rc}): {L.sg_last_error().decode()}")

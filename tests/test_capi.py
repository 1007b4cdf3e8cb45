"""C-ABI checks that need no GPU: libsg.so loads, exports every entry point
include/sg.h declares, and the Python binding table matches the header."""

from __future__ import annotations

import ctypes
import re

from conftest import REPO


def header_symbols() -> set[str]:
    text = (REPO / "include" / "sg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_header_symbol():
    lib = ctypes.CDLL(str(REPO / "paper_2210_06439_b200" / "libsg.so"))
    missing = [s for s in sorted(header_symbols()) if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sg_abi_version() == 2


def test_binding_table_covers_header():
    from paper_2210_06439_b200 import _lib
    declared = header_symbols() - {"sg_last_error"}
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    L = _lib.load()
    assert L.sg_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a_and_unfused():
    """The cubin targets sm_100a; the data path has no -use_fast_math."""
    mk = (REPO / "paper_2210_06439_b200" / "csrc" / "Makefile").read_text()
    assert "arch=compute_100a,code=sm_100a" in mk
    assert "-fmad=false" in mk and "fast_math" not in mk.replace("never -use_fast_math", "")


def test_no_cpu_fallback_without_device(monkeypatch):
    """On a host without CUDA the product path raises instead of computing."""
    import pytest
    import torch

    from paper_2210_06439_b200 import _lib, kernels, octree
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    tree = octree.build_unigrid(1)
    with pytest.raises(_lib.SGUnavailable):
        kernels.max_wavespeed(tree.leaves[0], kernels.HydroConfig())

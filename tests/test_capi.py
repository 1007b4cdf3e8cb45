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
    assert lib.sg_abi_version() == 4


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


def test_argument_validation_without_device():
    """Every entry point rejects NULL required pointers and bad geometry with
    SG_EINVAL naming the argument, before touching CUDA (so this runs on a
    host without a GPU); empty batches are no-ops."""
    import pytest

    from paper_2210_06439_b200 import _lib
    L = _lib.load()
    P = 4096  # stand-in device address: never dereferenced, validation fails first
    N = None
    d = 1.0 / 64

    def bad(name, *args, match):
        rc = getattr(L, name)(*args)
        msg = L.sg_last_error().decode()
        assert rc == 1, (name, rc, msg)
        assert match in msg, (name, msg)

    bad("sg_cluster_aggregate", N, 24, 24, 24, 1, d, P, N, match="mass is NULL")
    bad("sg_cluster_aggregate", P, 24, 24, 24, 1, d, N, N, match="clusters is NULL")
    bad("sg_cluster_aggregate", P, 23, 24, 24, 1, d, P, N, match="even")
    p2p = lambda **kw: [kw.get("mass", P), 8, 8, kw.get("nz", 8), kw.get("pad", 2), 0, N, 1, d, 1e-3, 1e-5,
                        kw.get("halo", 2), kw.get("out", P), 8, 8, 8, 0, kw.get("prec", 0), N]
    bad("sg_p2p", *p2p(mass=N), match="mass is NULL")
    bad("sg_p2p", *p2p(out=N), match="out is NULL")
    bad("sg_p2p", *p2p(halo=3), match="halo")
    bad("sg_p2p", *p2p(nz=-8), match="bad mass view")
    bad("sg_p2p", *p2p(prec=7), match="precision")
    m2l = lambda **kw: [kw.get("mass", P), 8, 8, 8, kw.get("pad", 8), 0, kw.get("cl", P), 0, N,
                        kw.get("nleaves", 1), d, 1e-3, 1e-5, kw.get("order", 1), 0, 512, kw.get("out", P),
                        8, 8, 8, 0, kw.get("ws", P), 1 << 40, kw.get("prec", 0), N]
    bad("sg_m2l", *m2l(mass=N), match="mass is NULL")
    bad("sg_m2l", *m2l(cl=N), match="clusters is NULL")
    bad("sg_m2l", *m2l(out=N), match="out is NULL")
    bad("sg_m2l", *m2l(pad=7), match="pad")
    bad("sg_m2l", *m2l(order=2), match="order")
    bad("sg_m2l", *m2l(prec=5), match="precision")
    bad("sg_m2l", *m2l(ws=N), match="workspace")
    assert L.sg_m2l(*m2l(mass=N, cl=N, out=N, ws=N, nleaves=0)) == 0
    bad("sg_reconstruct", N, 8, 8, 8, 2, 0, N, 1, 1e-12, P, N, match="U is NULL")
    bad("sg_reconstruct", P, 8, 8, 8, 2, 0, N, 1, 1e-12, N, N, match="Q is NULL")
    bad("sg_reconstruct", P, 8, 8, 8, 1, 0, N, 1, 1e-12, P, N, match="pad")
    for fn in ("sg_flux", "sg_flux_legacy"):
        bad(fn, N, 1, 1.4, P, P, P, P, P, N, N, 0, N, match="Q is NULL")
        bad(fn, P, 1, 1.4, N, P, P, P, P, N, N, 0, N, match="FX is NULL")
        bad(fn, P, 1, 1.4, P, P, P, N, P, N, N, 0, N, match="smax is NULL")
        bad(fn, P, 1, 1.4, P, P, P, P, N, N, N, 0, N, match="err is NULL")
        assert getattr(L, fn)(N, 0, 1.4, N, N, N, N, N, N, N, 0, N) == 0
    bad("sg_hydro_fused", N, 8, 8, 8, 2, 0, N, 1, 1e-12, 1.4, P, P, P, P, P, N, N, 0, N, match="U is NULL")
    bad("sg_hydro_fused", P, 8, 8, 8, 2, 0, N, 1, 1e-12, 1.4, P, P, N, P, P, N, N, 0, N, match="FZ is NULL")
    bad("sg_hydro_fused", P, 8, 8, 8, 1, 0, N, 1, 1e-12, 1.4, P, P, P, P, P, N, N, 0, N, match="pad")
    bad("sg_hydro_update", P, 8, 8, 8, 2, 0, N, 1, P, N, P, N, N, 1e-3, d, 0.4, N, N, N, 0, N, N,
        match="FY is NULL")
    bad("sg_hydro_update", P, -8, 8, 8, 2, 0, N, 1, P, P, P, N, N, 1e-3, d, 0.4, N, N, N, 0, N, N,
        match="bad U view")
    bad("sg_max_wavespeed", P, 8, 8, 8, 2, 0, N, 1, 1.4, 1e-12, N, N, match="smax is NULL")
    bad("sg_max_reduce", P, 3, N, N, match="out is NULL")
    bad("sg_max_reduce", N, 3, P, N, match="vals is NULL")
    bad("sg_dt_from_smax", P, 0.4, d, N, N, match="dt is NULL")
    bad("sg_fill_periodic", N, 1, 8, 8, 8, 2, 7, N, match="field is NULL")
    bad("sg_fill_periodic", P, 1, 8, 8, 8, -1, 7, N, match="bad geometry")
    bad("sg_gather_blocks", P, 8, 8, 8, 2, 0, N, 1, 1, 2, N, N, match="out is NULL")
    bad("sg_gather_blocks", P, 8, 8, 8, 2, 0, N, 1, 1, 3, P, N, match="halo")
    bad("sg_scale_copy", P, 8, N, 2, 8, 8, 8, 1.0, N, match="src is NULL")
    # per-subgrid drop-in entry points (host arrays): NULLs are rejected before any CUDA call
    bad("sg_dropin_max_wavespeed", N, 1.4, 1e-12, P, N, match="U is NULL")
    bad("sg_dropin_max_wavespeed", P, 1.4, 1e-12, N, N, match="smax is NULL")
    bad("sg_dropin_monopole", N, 2, d, 1e-3, 1e-5, 0, P, N, match="cube is NULL")
    bad("sg_dropin_monopole", P, 9, d, 1e-3, 1e-5, 0, P, N, match="halo")
    bad("sg_dropin_multipole", P, d, 1e-3, 1e-5, 1, 0, 512, 0, N, N, match="out is NULL")
    bad("sg_dropin_reconstruct", P, 1e-12, N, N, match="Q is NULL")
    bad("sg_dropin_flux", P, 1.4, P, P, P, P, N, N, match="err is NULL")
    bad("sg_dropin_hydro_update", N, P, P, P, 1e-3, d, 0.4, P, N, match="U is NULL")
    bad("sg_scale_copy", P, -1, P, 2, 8, 8, 8, 1.0, N, match="negative pad")
    flops = ctypes.c_int64()
    bad("sg_fp64_peak", 3, 1, P, ctypes.byref(flops), N, match="mode")
    bad("sg_fp64_peak", 0, 1, N, ctypes.byref(flops), N, match="sink is NULL")
    with pytest.raises(_lib.SGError, match="clusters is NULL"):
        _lib.call("sg_cluster_aggregate", P, 24, 24, 24, 1, d, N, N)

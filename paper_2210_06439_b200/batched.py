"""Batched device API: thin, allocation-free wrappers of the C ABI over torch
CUDA tensors (torch supplies device memory and the current stream only).

Every function launches asynchronously on ``torch.cuda.current_stream()``.
Field arguments follow the view convention of include/sg.h: a float64
tensor holding ``ncomp`` components of dims (nz+2p, ny+2p, nx+2p), plus the
interior dims, the pad and the leaf stride (0 for one global field).
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from dataclasses import dataclass

import torch

from . import _lib

U32_OK = 0xFFFFFFFF


def require_device() -> None:
    if not torch.cuda.is_available():
        raise _lib.SGUnavailable("no CUDA device: the sm_100a kernels have no CPU fallback")
    _lib.load()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must live on the CUDA device")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _f64(t):
    if t.dtype != torch.float64:
        raise TypeError(f"expected float64, got {t.dtype}")
    return _ptr(t)


@dataclass(frozen=True)
class View:
    """Interior dims + pad of a padded field (see include/sg.h)."""
    nx: int
    ny: int
    nz: int
    pad: int
    leaf_stride: int = 0

    @property
    def padded_shape(self) -> tuple[int, int, int]:
        p = 2 * self.pad
        return (self.nz + p, self.ny + p, self.nx + p)

    @property
    def volume(self) -> int:
        z, y, x = self.padded_shape
        return x * y * z


def cluster_aggregate(mass: torch.Tensor, dx: float, clusters: torch.Tensor, nleaf: int = 1) -> None:
    """mass (..., mnz, mny, mnx) -> clusters (..., mnz/2, mny/2, mnx/2, 4)."""
    mnz, mny, mnx = mass.shape[-3:]
    _lib.call("sg_cluster_aggregate", _f64(mass), mnx, mny, mnz, nleaf, float(dx), _f64(clusters), _stream())


def _prec(precision) -> int:
    if isinstance(precision, str):
        try:
            return _lib.PRECISIONS[precision]
        except KeyError:
            raise ValueError(f"precision must be one of {sorted(_lib.PRECISIONS)}, got {precision!r}") from None
    return int(precision)


def p2p(mass, mv: View, leaves, nleaves: int, dx: float, rad2: float, eps2: float, halo: int,
        out, ov: View, precision="exact") -> None:
    _lib.call("sg_p2p", _f64(mass), mv.nx, mv.ny, mv.nz, mv.pad, mv.leaf_stride, _ptr(leaves), nleaves,
              float(dx), float(rad2), float(eps2), int(halo), _f64(out), ov.nx, ov.ny, ov.nz,
              ov.leaf_stride, _prec(precision), _stream())


_WORKSPACE: "OrderedDict" = OrderedDict()
_WORKSPACE_LOCK = threading.Lock()
_WORKSPACE_MAX = 16  # (device, stream) entries kept; least recently used dropped


def m2l_workspace(nleaves: int, device=None) -> torch.Tensor:
    """Cached scratch for sg_m2l, one per (device, stream): callers on
    different streams (e.g. pool threads, SURVEY.md 8(b) re-entrancy) never
    share one; reuse on the same stream is stream-ordered.  Grows on demand;
    at most _WORKSPACE_MAX entries are kept (dropping one is safe: torch's
    caching allocator reuses a freed block only for its own stream)."""
    need = int(_lib.load().sg_m2l_workspace_bytes(nleaves))
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (dev, torch.cuda.current_stream(dev).cuda_stream)
    with _WORKSPACE_LOCK:
        ws = _WORKSPACE.get(key)
        if ws is None or ws.numel() * 8 < need:
            ws = torch.empty((need + 7) // 8, dtype=torch.float64, device=dev)
            _WORKSPACE[key] = ws
        _WORKSPACE.move_to_end(key)
        while len(_WORKSPACE) > _WORKSPACE_MAX:
            _WORKSPACE.popitem(last=False)
    return ws


def m2l(mass, mv: View, clusters, cluster_leaf_stride: int, leaves, nleaves: int, dx: float, rad2: float,
        eps2: float, order: int, out, ov: View, i0: int = 0, i1: int = 512, workspace=None,
        precision="exact") -> None:
    ws = workspace if workspace is not None else m2l_workspace(nleaves, mass.device)
    _lib.call("sg_m2l", _f64(mass), mv.nx, mv.ny, mv.nz, mv.pad, mv.leaf_stride, _f64(clusters),
              cluster_leaf_stride, _ptr(leaves), nleaves, float(dx), float(rad2), float(eps2), int(order),
              int(i0), int(i1), _f64(out), ov.nx, ov.ny, ov.nz, ov.leaf_stride, _f64(ws), ws.numel() * 8,
              _prec(precision), _stream())


def reconstruct(U, uv: View, leaves, nleaves: int, floor: float, Q) -> None:
    _lib.call("sg_reconstruct", _f64(U), uv.nx, uv.ny, uv.nz, uv.pad, uv.leaf_stride, _ptr(leaves),
              nleaves, float(floor), _f64(Q), _stream())


def flux(Q, nleaves: int, gamma: float, FX, FY, FZ, smax, err, latch=None, gate=None, it: int = 0) -> None:
    _lib.call("sg_flux", _f64(Q), nleaves, float(gamma), _f64(FX), _f64(FY), _f64(FZ), _f64(smax),
              _ptr(err), _ptr(latch), _ptr(gate), int(it), _stream())


def flux_legacy(Q, nleaves: int, gamma: float, FX, FY, FZ, smax, err, latch=None, gate=None,
                it: int = 0) -> None:
    """reference kernels/legacy.py flux formulation (not bitwise to flux())."""
    _lib.call("sg_flux_legacy", _f64(Q), nleaves, float(gamma), _f64(FX), _f64(FY), _f64(FZ), _f64(smax),
              _ptr(err), _ptr(latch), _ptr(gate), int(it), _stream())


def hydro_fused(U, uv: View, leaves, nleaves: int, floor: float, gamma: float, FX, FY, FZ, smax, err,
                latch=None, gate=None, it: int = 0) -> None:
    """reconstruct + flux without materialising Q (bit-identical outputs)."""
    _lib.call("sg_hydro_fused", _f64(U), uv.nx, uv.ny, uv.nz, uv.pad, uv.leaf_stride, _ptr(leaves), nleaves,
              float(floor), float(gamma), _f64(FX), _f64(FY), _f64(FZ), _f64(smax), _ptr(err), _ptr(latch),
              _ptr(gate), int(it), _stream())


def hydro_update(U, uv: View, leaves, nleaves: int, FX, FY, FZ, smax, dt_dev, dt: float, dx: float,
                 cfl: float, status, latch=None, gate=None, it: int = 0, err_info=None) -> None:
    _lib.call("sg_hydro_update", _f64(U), uv.nx, uv.ny, uv.nz, uv.pad, uv.leaf_stride, _ptr(leaves),
              nleaves, _f64(FX), _f64(FY), _f64(FZ), _ptr(smax), _ptr(dt_dev), float(dt), float(dx),
              float(cfl), _ptr(status), _ptr(latch), _ptr(gate), int(it), _ptr(err_info), _stream())


def max_wavespeed(U, uv: View, leaves, nleaves: int, gamma: float, pfloor: float, smax) -> None:
    _lib.call("sg_max_wavespeed", _f64(U), uv.nx, uv.ny, uv.nz, uv.pad, uv.leaf_stride, _ptr(leaves),
              nleaves, float(gamma), float(pfloor), _f64(smax), _stream())


def max_reduce(vals, n: int, out) -> None:
    _lib.call("sg_max_reduce", _f64(vals), n, _f64(out), _stream())


def dt_from_smax(s_pre, cfl: float, dx: float, dt) -> None:
    _lib.call("sg_dt_from_smax", _f64(s_pre), float(cfl), float(dx), _f64(dt), _stream())


def fill_periodic(field, ncomp: int, v: View, wrap_mask: int = 7) -> None:
    _lib.call("sg_fill_periodic", _f64(field), ncomp, v.nx, v.ny, v.nz, v.pad, int(wrap_mask), _stream())


def scale_copy(dst, dst_pad: int, src, src_pad: int, nx: int, ny: int, nz: int, scale: float) -> None:
    _lib.call("sg_scale_copy", _f64(dst), dst_pad, _f64(src), src_pad, nx, ny, nz, float(scale), _stream())


def gather_blocks(field, v: View, leaves, nleaves: int, ncomp: int, halo: int, out) -> None:
    """out[b, c] = the (8+2*halo)^3 box around leaf b (batched source_cube)."""
    _lib.call("sg_gather_blocks", _f64(field), v.nx, v.ny, v.nz, v.pad, v.leaf_stride, _ptr(leaves), nleaves,
              int(ncomp), int(halo), _f64(out), _stream())

"""Legacy hydro kernels on the B200: drop-in for
reference pkg/src/simdgrid/kernels/legacy.py (``legacy_reconstruct``,
``legacy_flux``), the straight-line kernels the paper's hydro comparison
(Fig. 6) runs against the vectorised ones.

The reference's legacy reconstruction computes exactly the values of the
production reconstruction (same slopes for every input incl. NaN, same
expression tree), so it runs ``sg_reconstruct``; the legacy flux has its own
formulation (``sg_flux_legacy``) and is bit-identical to legacy.py, physics-
equal (not bitwise) to the production flux.
"""

from __future__ import annotations

import numpy as np
import torch

from . import batched as B
from .kernels import FluxField, HydroConfig, KernelError, QuadratureField, _raise_flux_error, _to_dev, reconstruct

__all__ = ["legacy_reconstruct", "legacy_flux", "decode_legacy_flux_error", "KernelError"]


def legacy_reconstruct(sub, cfg: HydroConfig, backend=None) -> QuadratureField:
    """reference legacy.py:149-154 (``backend`` accepted and ignored)."""
    return reconstruct(sub, cfg, "scalar")


def decode_legacy_flux_error(err: int) -> tuple[int, int]:
    if err == B.U32_OK:
        return 0, -1
    return (err >> 10) & 3, err & 1023


def legacy_flux(sub, q: QuadratureField, cfg: HydroConfig, backend=None) -> FluxField:
    """reference legacy.py:157-167 (``backend`` accepted and ignored)."""
    dQ = q.device_values() if isinstance(q, QuadratureField) else None
    if dQ is None:
        dQ = _to_dev(q.values)
    dev = dQ.device
    FX = torch.empty((5, 8, 8, 9), dtype=torch.float64, device=dev)
    FY = torch.empty((5, 8, 9, 8), dtype=torch.float64, device=dev)
    FZ = torch.empty((5, 9, 8, 8), dtype=torch.float64, device=dev)
    status = torch.empty(2, dtype=torch.float64, device=dev)  # [smax, err word]: one readback
    B.flux_legacy(dQ, 1, cfg.gamma, FX, FY, FZ, status[0:1], status[1:2].view(torch.int32)[0:1])
    st = status.cpu().numpy()
    code, cell = decode_legacy_flux_error(int(st[1:2].view(np.uint32)[0]))
    if code != 0:
        _raise_flux_error(sub, code, cell)
    return FluxField(max_speed=float(st[0]), device_values=(FX, FY, FZ))


"""Backend-name registry accepted by the drop-in entry points.

The reference's kernels take a ``backend`` argument resolved through
``simd.get_backend`` (reference pkg/src/simdgrid/simd.py:428-452); it only
selects the CPU lane width W and results are bitwise W-independent.  The CUDA
kernels have no lane abstraction, so here the name is validated with the
same contract (unknown names and the unbuilt ``native`` backend raise
``BackendUnavailableError``) and otherwise ignored.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["Backend", "BackendUnavailableError", "available_backends", "get_backend", "lane_count"]


class BackendUnavailableError(ValueError):
    """Unknown or unbuilt backend name."""


@dataclass(frozen=True)
class Backend:
    name: str
    width: int


_REGISTRY = {"scalar": Backend("scalar", 1)}
for _w in (2, 4, 8, 16):
    _REGISTRY[f"emulated{_w}"] = Backend(f"emulated{_w}", _w)


def available_backends() -> tuple[str, ...]:
    return tuple(_REGISTRY)


def get_backend(backend) -> Backend:
    """Resolve a backend name; objects exposing ``name`` and ``width`` (e.g.
    the reference's own Backend instances) pass through."""
    if isinstance(backend, Backend) or (hasattr(backend, "width") and hasattr(backend, "name")):
        return backend
    if backend == "native":
        raise BackendUnavailableError(
            "the 'native' backend is not built in this installation; "
            f"available: {', '.join(available_backends())}")
    try:
        return _REGISTRY[backend]
    except (KeyError, TypeError):
        raise BackendUnavailableError(
            f"unknown backend {backend!r}; available: {', '.join(available_backends())}") from None


def lane_count(backend) -> int:
    return get_backend(backend).width

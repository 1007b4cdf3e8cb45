"""Profiler bridge: the reference's APEX-style
``Profiler`` API (reference pkg/src/simdgrid/profiling.py:30-86: ``timed``,
``region``, ``report``, ``total_ns``; records of count / total_ns / mean_ns)
measuring DEVICE time with CUDA events on the current stream instead of host
wall time, so the reference's reporting (CSV rows, plots) can consume GPU
kernel timings unchanged.

Events are only resolved in ``report()`` (one synchronisation), so timing
adds no host-device round trips inside the timed work.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass

__all__ = ["ProfileRecord", "CudaProfiler"]


@dataclass(frozen=True)
class ProfileRecord:
    name: str
    count: int
    total_ns: int

    @property
    def mean_ns(self) -> float:
        return self.total_ns / self.count


class CudaProfiler:
    """Device-time profiler.  ``weight`` lets one launch stand for several
    per-leaf evaluations (the reference counts one record per leaf job)."""

    def __init__(self):
        self._pending: list = []          # (name, start_event, end_event, weight)
        self._done: dict[str, tuple[int, int]] = {}

    def _events(self):
        import torch
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(self, name: str, work, weight: int = 1):
        """Run ``work()`` (which launches on the current stream), record its
        device time under ``name`` and pass the result through."""
        a, b = self._events()
        a.record()
        try:
            return work()
        finally:
            b.record()
            self._pending.append((name, a, b, weight))

    @contextmanager
    def region(self, name: str, weight: int = 1):
        a, b = self._events()
        a.record()
        try:
            yield
        finally:
            b.record()
            self._pending.append((name, a, b, weight))

    def add(self, name: str, count: int, total_ns: int) -> None:
        c, t = self._done.get(name, (0, 0))
        self._done[name] = (c + count, t + total_ns)

    def _resolve(self) -> None:
        if not self._pending:
            return
        import torch
        torch.cuda.synchronize()
        for name, a, b, w in self._pending:
            self.add(name, w, int(round(a.elapsed_time(b) * 1e6)))
        self._pending.clear()

    def report(self) -> tuple:
        """Snapshot of all records, ordered by name (reference semantics)."""
        self._resolve()
        return tuple(ProfileRecord(n, c, t) for n, (c, t) in sorted(self._done.items()))

    def total_ns(self, name: str) -> int:
        for rec in self.report():
            if rec.name == name:
                return rec.total_ns
        return 0

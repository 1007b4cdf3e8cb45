"""Shared pytest setup: the `gpu` marker, repo-root imports, golden loaders."""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA C-ABI path)")
    config.addinivalue_line("markers", "slow: long CPU-oracle case (still part of the default run)")


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def bitwise(a, b) -> bool:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def leaf_digests(level: int, out4: np.ndarray) -> dict:
    na = 1 << level
    d = {}
    for cz in range(na):
        for cy in range(na):
            for cx in range(na):
                blk = out4[:, cz * 8:(cz + 1) * 8, cy * 8:(cy + 1) * 8, cx * 8:(cx + 1) * 8]
                d["%d,%d,%d" % (cx, cy, cz)] = digest(blk)
    return d


def leaves_to_global(level: int, leaves: np.ndarray, per_leaf: np.ndarray) -> np.ndarray:
    """(B, C, 512) per-leaf interior blocks -> (C, n, n, n) global arrays."""
    n = 8 << level
    C = per_leaf.shape[1]
    g = np.empty((C, n, n, n))
    for b, (cx, cy, cz) in enumerate(leaves.tolist()):
        g[:, cz * 8:(cz + 1) * 8, cy * 8:(cy + 1) * 8, cx * 8:(cx + 1) * 8] = per_leaf[b].reshape(C, 8, 8, 8)
    return g


@pytest.fixture(scope="session")
def manifest():
    return json.loads((GOLDEN / "manifest.json").read_text())


def load_npz(name: str):
    return np.load(GOLDEN / name)

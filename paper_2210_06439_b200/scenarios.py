"""Seeded synthetic workloads for BASELINE.json configs 1-5.

Every generator returns global cell-centred fields indexed ``[z, y, x]`` with
cell ``i`` centred at ``(i + 0.5) * dx`` -- the layout the reference's
``SubGrid.cell_centers`` (reference pkg/src/simdgrid/octree.py:63-71) and
``tests/util.py:global_field`` (reference pkg/tests/util.py:70-76) imply.

The only transcendental functions involved (``sin`` for the polytrope,
``pow`` for the barotropic pressure, ``exp`` inside ``lognormal``) go through
the scalar C library, never numpy's runtime-dispatched SIMD loops, so the same
seed yields the same bits on any x86-64 host of this image (the golden
fixtures also record an input digest so a host that disagrees is detected).
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "cell_centres",
    "config1_cube",
    "config2_rho",
    "polytrope_rho",
    "config3_rho",
    "config4_state",
    "config5_state",
    "CONFIG5_FLOOR",
    "CONFIG5_OMEGA",
]

CONFIG5_FLOOR = 0.05   # reference STAR_ATMOSPHERE (scenarios.py:29); 1e-10 fails in the reference
CONFIG5_OMEGA = 0.1
POLYTROPE_RADIUS = 0.3


def _n(level: int) -> int:
    return 8 << level


def cell_centres(level: int) -> np.ndarray:
    """1-D centre coordinates ``(i + 0.5) * dx`` of a level-``level`` grid."""
    n = _n(level)
    dx = 1.0 / n
    return (np.arange(n, dtype=np.float64) + 0.5) * dx


def config1_cube(seed: int = 0) -> np.ndarray:
    """Config 1: one 24^3 mass neighbourhood, lognormal(0, 1)."""
    rng = np.random.default_rng(seed)
    return rng.lognormal(0.0, 1.0, (24, 24, 24))


def config2_rho(seed: int = 1, level: int = 3) -> np.ndarray:
    """Config 2: lognormal(0, 1) density on the 64^3 (level-3) unigrid."""
    rng = np.random.default_rng(seed)
    n = _n(level)
    return rng.lognormal(0.0, 1.0, (n, n, n))


def _radius_field(level: int) -> tuple[np.ndarray, np.ndarray]:
    """Return (r2, offsets): squared distance of every cell centre to the box
    centre (exact: dyadic offsets) and the per-axis offset vector."""
    c = cell_centres(level) - 0.5
    c2 = c * c
    r2 = (c2[:, None, None] + c2[None, :, None]) + c2[None, None, :]
    return r2, c


def polytrope_rho(level: int, floor: float, radius: float = POLYTROPE_RADIUS) -> np.ndarray:
    """n=1 polytrope rho = sin(pi r/R)/(pi r/R) for r < R, floored at ``floor``.

    sin is evaluated once per distinct r^2 with ``math.sin`` (scalar libm)."""
    r2, _ = _radius_field(level)
    uniq, inv = np.unique(r2, return_inverse=True)
    vals = np.empty_like(uniq)
    for k, v in enumerate(uniq.tolist()):
        r = math.sqrt(v)
        if r < radius:
            q = math.pi * r / radius
            rho = math.sin(q) / q
        else:
            rho = 0.0
        vals[k] = rho if rho > floor else floor
    return vals[inv].reshape(r2.shape)


def config3_rho(level: int = 3) -> np.ndarray:
    """Config 3: polytrope with the BASELINE floor 1e-10 (deterministic)."""
    return polytrope_rho(level, 1e-10)


def config4_state(level: int = 3) -> dict[str, np.ndarray]:
    """Config 4: Sedov-like state -- rho=1, s=0, E=1e-5, and total energy 1
    deposited uniformly in the central 2^3 cells (E = 1/(8 dx^3)).

    The centre selection mirrors the reference blast init
    (reference scenarios.py:70): |X-0.5| < dx on every axis."""
    n = _n(level)
    dx = 1.0 / n
    c = cell_centres(level)
    near = np.abs(c - 0.5) < dx
    centre = near[:, None, None] & near[None, :, None] & near[None, None, :]
    rho = np.ones((n, n, n))
    E = np.full((n, n, n), 1e-5)
    E[centre] = 1.0 / (8.0 * dx * dx * dx)
    z = np.zeros((n, n, n))
    return {"rho": rho, "sx": z, "sy": z.copy(), "sz": z.copy(), "E": E}


def config5_state(level: int = 4, gamma: float = 1.4,
                  floor: float = CONFIG5_FLOOR, omega: float = CONFIG5_OMEGA) -> dict[str, np.ndarray]:
    """Config 5: rotating polytrope, p = rho^gamma (K=1, reference
    scenarios.py:93), rigid rotation about z through the box centre."""
    rho = polytrope_rho(level, floor)
    _, c = _radius_field(level)
    n = _n(level)
    X = np.broadcast_to(c[None, None, :], (n, n, n))
    Y = np.broadcast_to(c[None, :, None], (n, n, n))
    vx = -omega * Y
    vy = omega * X
    uniq, inv = np.unique(rho, return_inverse=True)
    p = np.array([math.pow(v, gamma) for v in uniq.tolist()])[inv].reshape(rho.shape)
    E = p / (gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy)
    return {
        "rho": rho,
        "sx": rho * vx,
        "sy": rho * vy,
        "sz": np.zeros((n, n, n)),
        "E": E,
    }


# NaN injections for the error-path parity cases (tests/golden/make_golden.py
# "errors"): (z, y, x) global cells at level 2.  (4, 4, 30) sits one layer
# inside the +x face of leaf (3, 0, 0), whose periodic +x neighbour is leaf
# (0, 0, 0): minmod zeroes a NaN in the outer ghost layer, so that leaf only
# fails once the NaN has advanced one cell -- in hydro iteration 2.  (4, 12, 12)
# is the centre of leaf (1, 1, 0).  Morton keys: (0,0,0) 0 < (1,1,0) 3 < (3,0,0) 9.
ERROR_CASES = {
    "late_neighbour": ((4, 4, 30),),
    "two_leaves": ((4, 4, 30), (4, 12, 12)),
}


def config5_error_state(case: str, level: int = 2) -> dict[str, np.ndarray]:
    """config5_state(level) with rho = NaN at the ERROR_CASES[case] cells."""
    st = {k: np.array(v) for k, v in config5_state(level).items()}
    for z, y, x in ERROR_CASES[case]:
        st["rho"][z, y, x] = np.nan
    return st

"""Oracle vs the live reference on fresh seeded inputs (CPU; runs only where
the reference is importable -- the build container -- and is skipped on GPU
boxes).  Complements the committed fixtures (test_oracle_golden.py) with
parameters the fixtures do not pin: non-power-of-2 dx, other theta / eps /
gamma / floors, random [i0, i1) chunks, error-triggering hydro blocks.

The reference's compiled kernels are called exactly as its entry points call
them (reference kernels/__init__.py:122-267, compiled.py:31-480)."""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref():
    if not REF.is_dir():
        pytest.skip("reference package not present (GPU box)")
    pytest.importorskip("numba")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from simdgrid.kernels import compiled, geometry
    return compiled, geometry


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    oracle.build()
    return oracle


def same(a, b) -> bool:
    """bitwise, every NaN equal to every NaN (payloads are not specified)."""
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    na, nb = np.isnan(a), np.isnan(b)
    return bool(np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64), b[~nb].view(np.uint64)))


def hydro_block(rng, kind: int) -> np.ndarray:
    U = np.empty((5, 12, 12, 12))
    U[0] = rng.uniform(0.5, 2.0, (12, 12, 12))
    U[1:4] = rng.normal(0.0, 0.3, (3, 12, 12, 12))
    U[4] = rng.uniform(1.0, 3.0, (12, 12, 12))
    if kind == 1:    # strong gradients: floors and the energy fix-up engage
        U[0] *= rng.choice([1e-6, 1.0, 50.0], size=(12, 12, 12))
        U[1:4] *= 20.0
    return U


def poison(rng, Q: np.ndarray, kind: int) -> np.ndarray:
    """Reconstruction floors rho and E, so the flux error paths are reached
    the way the reference's tests reach them: an edited quadrature field.
    kind 2: a non-positive density (code 1); kind 3: E = 0 with momentum,
    i.e. non-positive pressure (code 2).  Several poisoned points, so the
    first one in the reference's loop order decides the reported cell."""
    Q = Q.copy()
    for _ in range(3):
        d, z, y, x = rng.integers(0, 26), rng.integers(1, 9), rng.integers(1, 9), rng.integers(1, 9)
        if kind == 2:
            Q[0, d, z, y, x] = -0.5
        elif kind == 3:
            Q[4, d, z, y, x] = 0.0
            Q[1, d, z, y, x] = 1.0
    return Q


@pytest.mark.parametrize("seed", range(8))
def test_hydro_kernels_match_reference(ref, O, seed):
    compiled, geo = ref
    rng = np.random.default_rng(1000 + seed)
    U = hydro_block(rng, seed % 4)
    floor = [1e-12, 0.05, 1e-3, 1e-9][seed % 4]
    gamma = [1.4, 5.0 / 3.0, 1.1 + 0.8 * rng.random(), 1.3][seed % 4]
    Qr = np.empty((5, 26, 10, 10, 10))
    compiled.reconstruct_kernel(U, floor, 1, geo.DIRECTIONS_F, Qr)
    Qo = O.reconstruct(U, floor)
    assert same(Qo, Qr)
    Qr = poison(rng, Qr, seed % 4)
    FX, FY, FZ = np.empty((5, 8, 8, 9)), np.empty((5, 8, 9, 8)), np.empty((5, 9, 8, 8))
    smax, code, cell = compiled.flux_kernel(Qr, gamma, 1, geo.DIR_PLUS, geo.DIR_MINUS, geo.SIMPSON_W, FX, FY, FZ)
    oFX, oFY, oFZ, osmax, ocode, ocell = O.flux(Qr, gamma)
    assert (ocode, ocell) == (int(code), int(cell))
    assert int(code) == {2: 1, 3: 2}.get(seed % 4, 0), (seed, code)
    assert same(oFX, FX) and same(oFY, FY) and same(oFZ, FZ) and same(osmax, smax)
    dtdx = float(rng.uniform(1e-3, 0.2))
    Ur = U.copy()
    compiled.hydro_update_kernel(Ur, FX, FY, FZ, dtdx)
    assert same(O.hydro_update(U, FX, FY, FZ, dtdx), Ur)
    pfloor = [1e-12, 1e-3][seed % 2]
    assert same(O.max_wavespeed(U, gamma, pfloor), compiled.max_wavespeed_kernel(U, gamma, pfloor))


GRAVITY_CASES = [  # (dx, theta, eps, order)
    (1.0 / 64, 0.34, 0.5, 1),
    (0.013, 0.34, 0.5, 0),
    (1.0 / 100, 0.22, 1.1, 1),
    (0.0371, 0.5, 0.3, 1),
    (1.0 / 128, 0.8, 0.5, 0),
    (0.02, 0.27, 0.75, 1),
]


@pytest.mark.parametrize("case", range(len(GRAVITY_CASES)))
def test_gravity_kernels_match_reference(ref, O, case):
    compiled, _ = ref
    dx, theta, eps, order = GRAVITY_CASES[case]
    rng = np.random.default_rng(2000 + case)
    cube = rng.lognormal(0.0, 1.0, (24, 24, 24)) * dx ** 3
    cube[rng.random((24, 24, 24)) < 0.03] = 0.0
    rad = dx / theta
    rad2 = rad * rad
    epsd = eps * dx
    eps2 = epsd * epsd
    # clusters + one random chunk [i0, i1) of the M2L, as multipole_prepare / run
    M, Dx, Dy, Dz = compiled.cluster_aggregate(cube, dx)
    oM, oDx, oDy, oDz = O.cluster_aggregate(cube, dx)
    assert same(oM, M) and same(oDx, Dx) and same(oDy, Dy) and same(oDz, Dz)
    i0 = int(rng.integers(0, 256))
    i1 = int(rng.integers(i0 + 1, 513))
    res = np.zeros((4, 8, 8, 8))
    compiled.multipole_kernel_impl(cube, M, Dx, Dy, Dz, dx, rad2, eps2, order, 1, i0, i1,
                                   res[0], res[1], res[2], res[3])
    assert same(O.multipole(cube, dx, theta, eps, order, i0, i1), res)
    # P2P on the central (8+2h)^3
    h = min(int(1.0 / theta), 8)
    sub = np.ascontiguousarray(cube[8 - h:16 + h, 8 - h:16 + h, 8 - h:16 + h])
    res = np.zeros((4, 8, 8, 8))
    compiled.monopole_kernel_impl(sub, dx, rad2, eps2, h, 1, res[0], res[1], res[2], res[3])
    assert same(O.monopole(sub, dx, theta, eps), res)

"""Randomised parity: CUDA path vs the CPU oracle (bit-pinned to the
reference by tests/test_oracle_golden.py) on seeded inputs outside the
fixtures -- non-power-of-two cell widths, varied theta / eps / order, varied
gamma / floor, NaN-poisoned inputs.  Bitwise (NaNs compared as NaNs)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import kernels as K  # noqa: E402
from paper_2210_06439_b200.batched import View  # noqa: E402


def same(a, b) -> bool:
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    na, nb = np.isnan(a), np.isnan(b)
    return a.shape == b.shape and np.array_equal(na, nb) and np.array_equal(a[~na].view(np.uint64),
                                                                             b[~nb].view(np.uint64))


CASES = [(1.0 / 64, 0.34, 0.5, 1), (0.1, 0.34, 0.5, 1), (1.0 / 3.0, 0.5, 0.25, 0), (7.0, 0.27, 1.5, 1),
         (1e-3, 0.34, 0.5, 0), (0.05, 0.2, 0.5, 1)]


@pytest.mark.parametrize("dx,theta,eps,order", CASES)
def test_m2l_p2p_random_cubes(dx, theta, eps, order):
    rng = np.random.default_rng(int(dx * 1e6) + int(theta * 100))
    cube = rng.lognormal(0.0, 1.0, (24, 24, 24)) * dx ** 3
    cube[rng.uniform(size=cube.shape) < 0.05] = 0.0
    d = torch.from_numpy(cube).cuda()
    cl = torch.empty((12, 12, 12, 4), dtype=torch.float64, device="cuda")
    B.cluster_aggregate(d, dx, cl)
    cfg = K.GravityConfig(theta=theta, eps=eps, expansion_order=order)
    rad2, eps2 = K.gravity_params(dx, cfg)
    out = torch.zeros((4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.m2l(d, View(8, 8, 8, 8), cl, 0, None, 1, dx, rad2, eps2, order, out, View(8, 8, 8, 0))
    assert same(out.cpu().numpy(), O.multipole(cube, dx, theta, eps, order))
    h = K.gravity_halo(theta)
    sub = np.ascontiguousarray(cube[8 - h:16 + h, 8 - h:16 + h, 8 - h:16 + h])
    out.zero_()
    B.p2p(torch.from_numpy(sub).cuda(), View(8, 8, 8, h), None, 1, dx, rad2, eps2, h, out, View(8, 8, 8, 0))
    assert same(out.cpu().numpy(), O.monopole(sub, dx, theta, eps))


@pytest.mark.parametrize("nb,dx", [(64, 1.0 / 64), (2400, 1.0 / 128), (64, 0.1)])
def test_p2p_batched_edge_masses_vs_oracle(nb, dx):
    """Batched P2P (the persistent TMA-staged stencil kernel: 64 subgrids in
    one partial round, 2400 in several rounds per CTA) bitwise against
    the oracle per subgrid, with cubes aimed at the exact K8 shortcut's
    guards: zeros (+/-), NaN, inf, subnormal and huge masses, masses at the
    edges of the shortcut's exponent range; dx = 0.1 (not a power of two)
    must take the plain 9-op loop."""
    rng = np.random.default_rng(nb)
    cubes = rng.lognormal(0.0, 1.0, (nb, 12, 12, 12)) * dx ** 3
    special = [np.nan, np.inf, -np.inf, 5e-324, 2.0 ** -1030, 2.0 ** -900, 2.0 ** -700, 2.0 ** 700,
               2.0 ** 900, 1e308, -0.0, 0.0]
    checked = list(range(0, nb, max(1, nb // 40)))
    for j, i in enumerate(checked):
        k = j % (len(special) + 4)
        if k < len(special):
            cubes[i, rng.integers(0, 12), rng.integers(0, 12), rng.integers(0, 12)] = special[k]
        elif k == len(special):
            cubes[i] *= -1.0                                   # negative masses
        elif k == len(special) + 1:
            cubes[i][rng.uniform(size=(12, 12, 12)) < 0.3] = -0.0
    d = torch.from_numpy(cubes).cuda()
    cfg = K.GravityConfig(theta=0.34, eps=0.5)
    rad2, eps2 = K.gravity_params(dx, cfg)
    out = torch.zeros((nb, 4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.p2p(d, View(8, 8, 8, 2, 12 ** 3), None, nb, dx, rad2, eps2, 2, out, View(8, 8, 8, 0, 4 * 512))
    got = out.cpu().numpy()
    for i in checked:
        assert same(got[i], O.monopole(cubes[i], dx, 0.34, 0.5)), i


def test_m2l_nan_and_inf_masses_propagate_like_reference():
    rng = np.random.default_rng(9)
    cube = rng.lognormal(0.0, 1.0, (24, 24, 24))
    cube[3, 4, 5] = np.nan        # a far cluster
    cube[12, 11, 12] = np.inf     # a near cell of central targets
    d = torch.from_numpy(cube).cuda()
    cl = torch.empty((12, 12, 12, 4), dtype=torch.float64, device="cuda")
    B.cluster_aggregate(d, 1.0 / 64, cl)
    rad2, eps2 = K.gravity_params(1.0 / 64, K.GravityConfig())
    out = torch.zeros((4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.m2l(d, View(8, 8, 8, 8), cl, 0, None, 1, 1.0 / 64, rad2, eps2, 1, out, View(8, 8, 8, 0))
    assert same(out.cpu().numpy(), O.multipole(cube, 1.0 / 64, 0.34, 0.5, 1))


@pytest.mark.parametrize("gamma,floor,seed", [(1.4, 1e-12, 1), (5.0 / 3.0, 1e-6, 2), (1.1, 1e-3, 3), (2.0, 1e-9, 4)])
def test_hydro_random_blocks(gamma, floor, seed):
    rng = np.random.default_rng(seed)
    nb = 8
    blocks = []
    for i in range(nb):
        scale = float(2.0 ** rng.integers(-8, 9)) * (1.0 + rng.uniform())
        rho = (1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))) * scale
        v = rng.uniform(-1, 1, (3, 12, 12, 12))
        p = (1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))) * scale
        U = np.stack([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * (v ** 2).sum(0)])
        if i == 5:
            U[4] *= 0.001          # energies clamped by the reconstruction floor
        if i == 6:
            U[0, 7, 3, 4] = np.nan  # poison reaches the interior
        blocks.append(U)
    Ud = torch.from_numpy(np.stack(blocks)).cuda()
    v = View(8, 8, 8, 2, leaf_stride=5 * 1728)
    Q = torch.empty((nb, 5, 26, 1000), dtype=torch.float64, device="cuda")
    B.reconstruct(Ud, v, None, nb, floor, Q)
    FX = torch.empty((nb, 5, 8, 8, 9), dtype=torch.float64, device="cuda")
    FY = torch.empty((nb, 5, 8, 9, 8), dtype=torch.float64, device="cuda")
    FZ = torch.empty((nb, 5, 9, 8, 8), dtype=torch.float64, device="cuda")
    smax = torch.empty(nb, dtype=torch.float64, device="cuda")
    err = torch.empty(nb, dtype=torch.int32, device="cuda")
    B.flux(Q, nb, gamma, FX, FY, FZ, smax, err)
    ws = torch.empty(nb, dtype=torch.float64, device="cuda")
    B.max_wavespeed(Ud, v, None, nb, gamma, floor, ws)
    Qh, FXh, FYh, FZh = (t.cpu().numpy() for t in (Q, FX, FY, FZ))
    for i, U in enumerate(blocks):
        Qw = O.reconstruct(U, floor)
        assert same(Qh[i].reshape(Qw.shape), Qw), i
        fx, fy, fz, s, code, cell = O.flux(Qw, gamma)
        assert same(FXh[i], fx) and same(FYh[i], fy) and same(FZh[i], fz), i
        assert K.decode_flux_error(int(err[i].cpu().numpy().view(np.uint32))) == (code, cell), i
        assert same(smax[i].item(), s) and same(ws[i].item(), O.max_wavespeed(U, gamma, floor)), i
    # fused path on the same blocks: fluxes, smax and first error
    FX2, FY2, FZ2 = torch.empty_like(FX), torch.empty_like(FY), torch.empty_like(FZ)
    smax2, err2 = torch.empty_like(smax), torch.empty_like(err)
    B.hydro_fused(Ud, v, None, nb, floor, gamma, FX2, FY2, FZ2, smax2, err2)
    assert same(FX2.cpu().numpy(), FXh) and same(FY2.cpu().numpy(), FYh) and same(FZ2.cpu().numpy(), FZh)
    assert same(smax2.cpu().numpy(), smax.cpu().numpy())
    assert np.array_equal(err2.cpu().numpy(), err.cpu().numpy())


def _edge_blocks(gamma):
    """Hydro blocks with the values exact arithmetic shortcuts get wrong
    (DESIGN.md 9.2 measured two for the fused kernel): -0.0 centre values
    under zero slopes (the zero-sum sign reaches u + 0.5*sum), +0.0
    momenta, infinite slopes, and magnitudes outside 2^+-500 / subnormal."""
    rng = np.random.default_rng(77)
    out = []
    for kind in range(8):
        rho = 1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))
        v = rng.uniform(-1, 1, (3, 12, 12, 12))
        p = 1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))
        U = np.stack([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * (v ** 2).sum(0)])
        if kind == 0:                     # uniform state, momenta all -0.0
            U[0], U[4] = 1.0, 2.5
            U[1:4] = -0.0
        elif kind == 1:                   # -0.0 momenta in a constant patch, random elsewhere
            U[:, 3:9, 3:9, 3:9] = np.array([1.0, -0.0, -0.0, -0.0, 2.5])[:, None, None, None]
        elif kind == 2:                   # mixed +0.0 / -0.0 momenta on a uniform background
            U[0], U[4] = 1.0, 2.5
            U[1:4] = np.where(rng.uniform(size=(3, 12, 12, 12)) < 0.5, 0.0, -0.0)
        elif kind == 3:                   # an infinite energy: infinite slopes around it
            U[4, 6, 5, 6] = np.inf
        elif kind == 4:                   # huge scale: exponents beyond 2^500
            U *= 2.0 ** 700
        elif kind == 5:                   # tiny scale: beyond 2^-500
            U *= 2.0 ** -700
        elif kind == 6:                   # subnormal momenta
            U[1:4] *= 2.0 ** -1070
        elif kind == 7:                   # -0.0 densities and energies in a uniform patch
            U[:, 2:6, 2:6, 2:6] = np.array([-0.0, 0.3, -0.0, 0.1, -0.0])[:, None, None, None]
        out.append(U)
    return np.stack(out)


@pytest.mark.parametrize("floor", [0.0, 1e-12])
def test_fused_hydro_edge_values_vs_oracle(floor):
    """The deduplicated fused kernel bitwise against the oracle on the edge
    blocks (fluxes, smax, first-error word)."""
    gamma = 1.4
    U = _edge_blocks(gamma)
    nb = len(U)
    Ud = torch.from_numpy(U).cuda()
    v = View(8, 8, 8, 2, leaf_stride=5 * 1728)
    shp = dict(dtype=torch.float64, device="cuda")
    F = [torch.empty((nb, 5, 8, 8, 9), **shp), torch.empty((nb, 5, 8, 9, 8), **shp),
         torch.empty((nb, 5, 9, 8, 8), **shp)]
    s = torch.empty(nb, **shp)
    e = torch.empty(nb, dtype=torch.int32, device="cuda")
    B.hydro_fused(Ud, v, None, nb, floor, gamma, *F, s, e)
    Fh = [f.cpu().numpy() for f in F]
    for i in range(nb):
        fx, fy, fz, sm, code, cell = O.flux(O.reconstruct(U[i], floor), gamma)
        assert K.decode_flux_error(int(e[i].cpu().numpy().view(np.uint32))) == (code, cell), i
        if code == 0:  # on an error the reference discards the outputs
            assert same(Fh[0][i], fx) and same(Fh[1][i], fy) and same(Fh[2][i], fz), i
            assert same(s[i].item(), sm), i


def _error_blocks(nb, seed, gamma):
    """nb random hydro blocks; every 7th one poisoned so the flux raises:
    negative pressure (code 2), non-positive density (code 1, needs
    floor <= 0), NaN, several errors in one block (first-error order)."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(nb):
        rho = 1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))
        v = rng.uniform(-1, 1, (3, 12, 12, 12))
        p = 1.0 + 0.5 * rng.uniform(-1, 1, (12, 12, 12))
        U = np.stack([rho, rho * v[0], rho * v[1], rho * v[2], p / (gamma - 1.0) + 0.5 * rho * (v ** 2).sum(0)])
        kind = i % 7
        z, y, x = rng.integers(1, 11, 3)
        if kind == 1:                       # kinetic energy above total energy: p < 0
            U[1, z, y, x] = 50.0
        elif kind == 2:                     # negative density (floor 0 keeps it)
            U[0, z, y, x] = -0.5
        elif kind == 3:
            U[0, z, y, x] = np.nan
        elif kind == 4:                     # two faults, the lower key wins
            U[1, z, y, x] = 50.0
            U[0, 11 - z, 11 - y, 11 - x] = -0.5
        elif kind == 5 and i % 2:           # fault on the ring only (ghost cell)
            U[2, 0, y, x] = 80.0
        out.append(U)
    return np.stack(out)


@pytest.mark.parametrize("nb,floor", [(40, 0.0), (333, 0.0), (333, 1e-12)])
def test_fused_hydro_errors_match_unfused(nb, floor):
    """The deduplicated fused kernel against reconstruct + flux (checked
    bitwise against the oracle above) on batches with poisoned blocks:
    fluxes, smax and the first-error word for every leaf, including batches
    larger than the persistent grid (several leaves per CTA, error flush at
    leaf boundaries)."""
    gamma = 1.4
    U = _error_blocks(nb, 11 + nb, gamma)
    Ud = torch.from_numpy(U).cuda()
    v = View(8, 8, 8, 2, leaf_stride=5 * 1728)
    Q = torch.empty((nb, 5, 26, 1000), dtype=torch.float64, device="cuda")
    shp = dict(dtype=torch.float64, device="cuda")
    F1 = [torch.empty((nb, 5, 8, 8, 9), **shp), torch.empty((nb, 5, 8, 9, 8), **shp),
          torch.empty((nb, 5, 9, 8, 8), **shp)]
    F2 = [torch.empty_like(f) for f in F1]
    s1, s2 = torch.empty(nb, **shp), torch.empty(nb, **shp)
    e1 = torch.empty(nb, dtype=torch.int32, device="cuda")
    e2 = torch.empty_like(e1)
    B.reconstruct(Ud, v, None, nb, floor, Q)
    B.flux(Q, nb, gamma, *F1, s1, e1)
    B.hydro_fused(Ud, v, None, nb, floor, gamma, *F2, s2, e2)
    e1h, e2h = e1.cpu().numpy(), e2.cpu().numpy()
    if floor == 0.0:  # a positive floor clamps every state: no error can occur
        assert (e1h.view(np.uint32) != B.U32_OK).sum() >= nb // 7, "too few error leaves"
    assert np.array_equal(e1h, e2h)
    assert same(s1.cpu().numpy(), s2.cpu().numpy())
    for a, b in zip(F1, F2):
        assert same(a.cpu().numpy(), b.cpu().numpy())


def test_acceptance_c1_hundred_random_subgrids_all_kernels():
    """Reference tests/test_acceptance.py:52-97 (c1) on the CUDA path: 100
    random subgrids through every array kernel in one stacked (drop-in
    layout) batch each -- cluster aggregation + M2L and P2P on random 24^3
    mass neighbourhoods (U(0,1) dx^3, 5% zeros; tests/util.py:43-50), and
    reconstruct, flux, update and max wave speed on gentle random states with
    a random power-of-two scale (tests/util.py:16-30) -- bitwise against the
    oracle, subgrid by subgrid."""
    rng = np.random.default_rng(4242)
    nb = 100
    dx = 1.0 / 64
    cfg = K.GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    rad2, eps2 = K.gravity_params(dx, cfg)
    cubes = rng.uniform(0.0, 1.0, (nb, 24, 24, 24))
    cubes[rng.uniform(size=cubes.shape) < 0.05] = 0.0
    cubes *= dx ** 3
    d = torch.from_numpy(cubes).cuda()
    cl = torch.empty((nb, 12, 12, 12, 4), dtype=torch.float64, device="cuda")
    B.cluster_aggregate(d, dx, cl, nb)
    m2l = torch.zeros((nb, 4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.m2l(d, View(8, 8, 8, 8, leaf_stride=24 ** 3), cl, 12 ** 3 * 4, None, nb, dx, rad2, eps2, 1, m2l,
          View(8, 8, 8, 0, leaf_stride=4 * 512))
    h = K.gravity_halo(cfg.theta)
    sub = np.ascontiguousarray(cubes[:, 8 - h:16 + h, 8 - h:16 + h, 8 - h:16 + h])
    S = 8 + 2 * h
    p2p = torch.zeros((nb, 4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.p2p(torch.from_numpy(sub).cuda(), View(8, 8, 8, h, leaf_stride=S ** 3), None, nb, dx, rad2, eps2, h, p2p,
          View(8, 8, 8, 0, leaf_stride=4 * 512))
    clh, m2lh, p2ph = cl.cpu().numpy(), m2l.cpu().numpy(), p2p.cpu().numpy()
    for i in range(nb):
        M, Dx, Dy, Dz = O.cluster_aggregate(cubes[i], dx)
        assert same(clh[i], np.stack([M, Dx, Dy, Dz], axis=-1)), i
        assert same(m2lh[i], O.multipole(cubes[i], dx, 0.34, 0.5, 1)), i
        assert same(p2ph[i], O.monopole(sub[i], dx, 0.34, 0.5)), i
    # hydro
    scale = 2.0 ** rng.integers(-4, 5, nb)
    U = np.empty((nb, 5, 12, 12, 12))
    U[:, 0] = rng.uniform(0.5, 1.5, (nb, 12, 12, 12))
    U[:, 1:4] = rng.normal(0.0, 0.1, (nb, 3, 12, 12, 12))
    U[:, 4] = rng.uniform(2.0, 3.0, (nb, 12, 12, 12))
    U *= scale[:, None, None, None, None]
    gamma, floor = 1.4, 1e-12
    dU = torch.from_numpy(U).cuda()
    v = View(8, 8, 8, 2, leaf_stride=5 * 1728)
    Q = torch.empty((nb, 5, 26, 1000), dtype=torch.float64, device="cuda")
    B.reconstruct(dU, v, None, nb, floor, Q)
    FX = torch.empty((nb, 5, 8, 8, 9), dtype=torch.float64, device="cuda")
    FY = torch.empty((nb, 5, 8, 9, 8), dtype=torch.float64, device="cuda")
    FZ = torch.empty((nb, 5, 9, 8, 8), dtype=torch.float64, device="cuda")
    smax = torch.empty(nb, dtype=torch.float64, device="cuda")
    err = torch.empty(nb, dtype=torch.int32, device="cuda")
    B.flux(Q, nb, gamma, FX, FY, FZ, smax, err)
    ws = torch.empty(nb, dtype=torch.float64, device="cuda")
    B.max_wavespeed(dU, v, None, nb, gamma, floor, ws)
    dtdx = 0.05
    st = torch.empty(nb, dtype=torch.int32, device="cuda")
    B.hydro_update(dU, v, None, nb, FX, FY, FZ, None, None, dtdx * dx, dx, 1e9, st)
    Qh, FXh, FYh, FZh = Q.cpu().numpy(), FX.cpu().numpy(), FY.cpu().numpy(), FZ.cpu().numpy()
    smh, errh, wsh, Uh = smax.cpu().numpy(), err.cpu().numpy().view(np.uint32), ws.cpu().numpy(), dU.cpu().numpy()
    for i in range(nb):
        q = O.reconstruct(U[i], floor)
        assert same(Qh[i].reshape(q.shape), q), i
        fx, fy, fz, s, code, cell = O.flux(q, gamma)
        assert same(FXh[i], fx) and same(FYh[i], fy) and same(FZh[i], fz) and smh[i] == s, i
        assert K.decode_flux_error(int(errh[i])) == ((0, -1) if code == 0 else (code, cell)), i
        assert wsh[i] == O.max_wavespeed(U[i], gamma, floor), i
        assert same(Uh[i], O.hydro_update(U[i], fx, fy, fz, dtdx)), i

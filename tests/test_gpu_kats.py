"""The reference's kernel contract tests (reference pkg/tests/test_gravity_kernels.py,
test_hydro_kernels.py, test_reference_kernels.py) ported to the drop-in API,
which runs them on the sm_100a kernels.  Known-answer tests, brute-force
oracles (numpy restatements of reference tests/util.py:82-146), symmetry,
error messages, NaN-poisoned stencil coverage, and backend-name invariance."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2210_06439_b200 import simd  # noqa: E402
from paper_2210_06439_b200.kernels import (FluxField, GravityConfig, HydroConfig, KernelError,  # noqa: E402
                                           flux, gravity_halo, hydro_update, max_wavespeed, monopole_kernel,
                                           multipole_kernel, multipole_prepare, reconstruct)
from paper_2210_06439_b200.octree import (EXT, HYDRO_FIELDS, SubGrid, build_unigrid,  # noqa: E402
                                          exchange_ghosts, neighborhood27, source_cube)

GAMMA = 1.4
BACKENDS = ["scalar", "emulated2", "emulated4", "emulated8", "emulated16"]


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def maxnorm_rel(got, want):
    return float(np.max(np.abs(got - want))) / float(np.max(np.abs(want)))


# -- fixtures (reference tests/util.py:16-55) ------------------------------------

def random_hydro_subgrid(rng, dx=1.0 / 64):
    sub = SubGrid.allocate(0, (0, 0, 0), dx)
    scale = float(2.0 ** rng.integers(-6, 7))
    shape = (EXT, EXT, EXT)
    rho = (1.0 + 0.1 * rng.uniform(-1.0, 1.0, shape)) * scale
    v = 0.1 * rng.uniform(-1.0, 1.0, (3, *shape))
    p = (1.0 + 0.1 * rng.uniform(-1.0, 1.0, shape)) * scale
    sub.fields["rho"][...] = rho
    sub.fields["sx"][...] = rho * v[0]
    sub.fields["sy"][...] = rho * v[1]
    sub.fields["sz"][...] = rho * v[2]
    sub.fields["E"][...] = p / (GAMMA - 1.0) + 0.5 * rho * (v ** 2).sum(axis=0)
    return sub


def uniform_subgrid(rho=1.0, v=(0.0, 0.0, 0.0), p=1.0, dx=1.0 / 64):
    sub = SubGrid.allocate(0, (0, 0, 0), dx)
    sub.fields["rho"][...] = rho
    sub.fields["sx"][...] = rho * v[0]
    sub.fields["sy"][...] = rho * v[1]
    sub.fields["sz"][...] = rho * v[2]
    sub.fields["E"][...] = p / (GAMMA - 1.0) + 0.5 * rho * (v[0] ** 2 + v[1] ** 2 + v[2] ** 2)
    return sub


def random_mass_tree(rng, level=1):
    tree = build_unigrid(level)
    for leaf in tree.leaves:
        m = rng.uniform(0.0, 1.0, (8, 8, 8))
        m[rng.uniform(size=(8, 8, 8)) < 0.05] = 0.0
        leaf.interior("mass")[...] = m * leaf.dx ** 3
    return tree


def gravity_setup(rng, level=1):
    tree = random_mass_tree(rng, level)
    return tree.leaves[0], neighborhood27(tree, 0)


def zero_mass_tree():
    tree = build_unigrid(1)
    for leaf in tree.leaves:
        leaf.interior("mass")[...] = 0.0
    return tree


def monopole_direct_sum(cube, dx, theta, eps, halo):
    rad2 = (dx / theta) ** 2
    eps2 = (eps * dx) ** 2
    out = [np.zeros((8, 8, 8)) for _ in range(4)]
    for oz in range(-halo, halo + 1):
        for oy in range(-halo, halo + 1):
            for ox in range(-halo, halo + 1):
                if (oz, oy, ox) == (0, 0, 0):
                    continue
                rx, ry, rz = -ox * dx, -oy * dx, -oz * dx
                r2 = rx * rx + ry * ry + rz * rz
                if r2 > rad2:
                    continue
                m = cube[halo + oz:halo + oz + 8, halo + oy:halo + oy + 8, halo + ox:halo + ox + 8]
                rt = np.sqrt(r2 + eps2)
                out[0] -= m / rt
                out[1] -= m * rx / rt ** 3
                out[2] -= m * ry / rt ** 3
                out[3] -= m * rz / rt ** 3
    return out


def gravity_full_direct_sum(cube, dx, eps):
    eps2 = (eps * dx) ** 2
    phi = np.zeros((8, 8, 8))

    def spans(o):
        return max(0, -8 - o), min(8, 16 - o)

    for oz in range(-15, 16):
        zlo, zhi = spans(oz)
        if zlo >= zhi:
            continue
        for oy in range(-15, 16):
            ylo, yhi = spans(oy)
            if ylo >= yhi:
                continue
            for ox in range(-15, 16):
                xlo, xhi = spans(ox)
                if xlo >= xhi or (oz, oy, ox) == (0, 0, 0):
                    continue
                r2 = (ox * dx) ** 2 + (oy * dx) ** 2 + (oz * dx) ** 2
                m = cube[zlo + oz + 8:zhi + oz + 8, ylo + oy + 8:yhi + oy + 8, xlo + ox + 8:xhi + ox + 8]
                phi[zlo:zhi, ylo:yhi, xlo:xhi] -= m / np.sqrt(r2 + eps2)
    return phi


# -- gravity (reference test_gravity_kernels.py) -------------------------------------

class TestMonopole:
    def test_single_source_at_one_cell_distance(self):
        tree = zero_mass_tree()
        target = tree.leaves[0]
        dx = target.dx
        target.interior("mass")[4, 4, 5] = 1.0
        phi, gx, gy, gz = monopole_kernel(target, neighborhood27(tree, 0), GravityConfig(theta=1.0, eps=1e-8))
        assert abs(phi[4, 4, 4] - (-1.0 / dx)) < 1e-6 / dx
        assert gx[4, 4, 4] > 0.0

    def test_self_interaction_masked_out(self):
        tree = zero_mass_tree()
        target = tree.leaves[0]
        target.interior("mass")[3, 3, 3] = 5.0
        phi, gx, gy, gz = monopole_kernel(target, neighborhood27(tree, 0), GravityConfig(theta=1.0))
        assert phi[3, 3, 3] == 0.0 and gx[3, 3, 3] == 0.0

    @pytest.mark.parametrize("theta", [0.5, 0.34, 0.2])
    def test_matches_direct_sum_oracle(self, theta):
        rng = np.random.default_rng(int(theta * 1000))
        target, sources = gravity_setup(rng)
        cfg = GravityConfig(theta=theta, eps=0.5)
        got = monopole_kernel(target, sources, cfg, "emulated8")
        halo = gravity_halo(theta)
        want = monopole_direct_sum(source_cube(sources, "mass", halo), target.dx, theta, cfg.eps, halo)
        for a, b in zip(got, want):
            assert maxnorm_rel(a, b) <= 1e-13

    def test_mirror_symmetry(self):
        tree = zero_mass_tree()
        target = tree.leaves[0]
        target.interior("mass")[4, 4, 1] = 2.0
        target.interior("mass")[4, 4, 6] = 2.0
        phi, *_ = monopole_kernel(target, neighborhood27(tree, 0), GravityConfig(theta=0.34))
        assert maxnorm_rel(phi[:, :, ::-1], phi) <= 1e-13

    @pytest.mark.parametrize("backend", BACKENDS[1:])
    def test_backend_matches_scalar_bitwise(self, backend):
        rng = np.random.default_rng(77)
        target, sources = gravity_setup(rng)
        ref = [a.copy() for a in monopole_kernel(target, sources, GravityConfig(), "scalar")]
        got = monopole_kernel(target, sources, GravityConfig(), backend)
        for a, b in zip(got, ref):
            assert np.array_equal(bits(a), bits(b))

    def test_requires_27_sources(self):
        tree = zero_mass_tree()
        with pytest.raises(ValueError, match="27"):
            monopole_kernel(tree.leaves[0], tree.leaves[:3], GravityConfig())

    def test_unknown_backend_rejected(self):
        tree = zero_mass_tree()
        with pytest.raises(simd.BackendUnavailableError, match="native"):
            monopole_kernel(tree.leaves[0], neighborhood27(tree, 0), GravityConfig(), "native")


class TestMultipole:
    def test_single_mass_far_cluster_equals_centroid_point(self):
        tree = zero_mass_tree()
        target = tree.leaves[0]
        dx = target.dx
        m = 3.0
        target.interior("mass")[6, 6, 6] = m
        cfg = GravityConfig(theta=1.0, eps=0.5, expansion_order=0)
        phi, *_ = multipole_kernel(target, neighborhood27(tree, 0), cfg)
        r2 = 3.0 * ((0.5 - 7.0) * dx) ** 2
        expect = -(m / np.sqrt(r2 + (cfg.eps * dx) ** 2))
        assert abs(phi[0, 0, 0] - expect) <= 1e-15 * abs(expect)

    def test_chunking_bitwise_invariant(self):
        rng = np.random.default_rng(88)
        target, sources = gravity_setup(rng)
        cfg = GravityConfig(expansion_order=1)
        ref = [a.copy() for a in multipole_kernel(target, sources, cfg, "emulated4", n_tasks=1)]
        for n in (16, 7):
            got = multipole_kernel(target, sources, cfg, "emulated4", n_tasks=n)
            for a, b in zip(got, ref):
                assert np.array_equal(bits(a), bits(b))

    def test_rejects_bad_n_tasks(self):
        target, sources = gravity_setup(np.random.default_rng(1))
        with pytest.raises(ValueError, match="n_tasks"):
            multipole_kernel(target, sources, GravityConfig(), "scalar", n_tasks=0)

    def test_error_decreases_with_theta(self):
        target, sources = gravity_setup(np.random.default_rng(99))
        full = gravity_full_direct_sum(source_cube(sources, "mass", 8), target.dx, 0.5)
        errs = {}
        for theta in (0.5, 0.34, 0.2):
            phi, *_ = multipole_kernel(target, sources, GravityConfig(theta=theta, eps=0.5), "emulated8")
            errs[theta] = float(np.max(np.abs(phi - full) / np.abs(full)))
        assert errs[0.5] > errs[0.34] > errs[0.2]

    def test_dipole_improves_on_monopole_expansion(self):
        rng = np.random.default_rng(1234)
        for _ in range(5):
            target, sources = gravity_setup(rng)
            full = gravity_full_direct_sum(source_cube(sources, "mass", 8), target.dx, 0.5)
            errs = {}
            for p in (0, 1):
                phi, *_ = multipole_kernel(target, sources, GravityConfig(expansion_order=p), "emulated8")
                errs[p] = float(np.max(np.abs(phi - full) / np.abs(full)))
            assert errs[1] <= errs[0]

    @pytest.mark.parametrize("backend", BACKENDS[1:])
    def test_backend_matches_scalar_bitwise(self, backend):
        target, sources = gravity_setup(np.random.default_rng(555))
        cfg = GravityConfig(expansion_order=1)
        ref = [a.copy() for a in multipole_kernel(target, sources, cfg, "scalar")]
        got = multipole_kernel(target, sources, cfg, backend)
        for a, b in zip(got, ref):
            assert np.array_equal(bits(a), bits(b))

    def test_prepare_chunks_cover_range(self):
        target, sources = gravity_setup(np.random.default_rng(10))
        cfg = GravityConfig()
        ref = [a.copy() for a in multipole_kernel(target, sources, cfg, "emulated8")]
        for a in (target.interior("phi"), target.interior("gx")):
            a[...] = 0.0
        run = multipole_prepare(target, sources, cfg, "emulated8")
        run(0, 100)
        run(100, 512)
        got = [target.interior(n) for n in ("phi", "gx", "gy", "gz")]
        for a, b in zip(got, ref):
            assert np.array_equal(bits(a), bits(b))


# -- hydro (reference test_hydro_kernels.py) -------------------------------------------

def euler_flux(rho, v, p, E, axis):
    vn = v[axis]
    f = [rho * vn, rho * v[0] * vn, rho * v[1] * vn, rho * v[2] * vn, (E + p) * vn]
    f[1 + axis] += p
    return f


class TestReconstruct:
    def test_uniform_gives_constant(self):
        sub = uniform_subgrid(rho=2.0, v=(0.1, -0.2, 0.3), p=1.5)
        q = reconstruct(sub, HydroConfig(), "emulated4")
        for v, name in enumerate(HYDRO_FIELDS):
            assert np.all(q.values[v] == sub.fields[name][2, 2, 2]), name

    def test_linear_ramp_unit_slopes(self):
        sub = uniform_subgrid(rho=1.0, p=1.0, dx=1.0)
        base = np.arange(EXT, dtype=np.float64)
        Z, Y, X = np.meshgrid(base, base, base, indexing="ij")
        ramp = X + Y + Z
        probe = (3, 2, 4)
        shift = 5.0 - ramp[probe[2] + 2, probe[1] + 2, probe[0] + 2]
        sub.fields["rho"][...] = ramp + shift
        q = reconstruct(sub, HydroConfig(), "scalar")
        assert q.value(0, probe, (1, 1, 0)) == 6.0
        assert q.value(0, probe, (-1, -1, 0)) == 4.0
        assert q.value(0, probe, (1, 1, 1)) == 6.5

    def test_positivity_floor_on_rho(self):
        cfg = HydroConfig()
        sub = uniform_subgrid(rho=1.0, p=1.0)
        base = np.arange(EXT, dtype=np.float64)
        Z, Y, X = np.meshgrid(base, base, base, indexing="ij")
        sub.fields["rho"][...] = 1e-6 * 4.0 ** (X + Y + Z)
        q = reconstruct(sub, cfg, "scalar")
        assert np.all(q.values[0] >= cfg.positivity_floor)
        assert q.values[0].min() == cfg.positivity_floor

    def test_positive_whenever_inputs_positive(self):
        rng = np.random.default_rng(11)
        for _ in range(5):
            q = reconstruct(random_hydro_subgrid(rng), HydroConfig(), "emulated8")
            assert np.all(q.values[0] > 0.0) and np.all(q.values[4] > 0.0)

    def test_reconstructed_pressure_positive(self):
        rng = np.random.default_rng(12)
        cfg = HydroConfig()
        sub = random_hydro_subgrid(rng)
        sub.fields["E"][...] *= 0.01
        q = reconstruct(sub, cfg, "scalar")
        ke = 0.5 * (q.values[1] ** 2 + q.values[2] ** 2 + q.values[3] ** 2) / q.values[0]
        assert np.all((cfg.gamma - 1.0) * (q.values[4] - ke) > 0.0)

    @pytest.mark.parametrize("backend", BACKENDS[1:])
    def test_backend_matches_scalar_bitwise(self, backend):
        sub = random_hydro_subgrid(np.random.default_rng(21))
        ref = reconstruct(sub, HydroConfig(), "scalar").values
        got = reconstruct(sub, HydroConfig(), backend).values
        assert np.array_equal(bits(got), bits(ref))

    def test_unfilled_ghost_sentinel(self):
        tree = build_unigrid(0, lambda X, Y, Z, dx: {"rho": np.ones_like(X)})
        with pytest.raises(KernelError, match="unfilled"):
            reconstruct(tree.leaves[0], HydroConfig(), "scalar", check_ghosts=True)


class TestFlux:
    def test_uniform_state_consistency(self):
        rho, v, p = 1.3, (0.4, -0.2, 0.1), 0.9
        sub = uniform_subgrid(rho=rho, v=v, p=p)
        E = p / (GAMMA - 1.0) + 0.5 * rho * sum(c * c for c in v)
        cfg = HydroConfig()
        fl = flux(sub, reconstruct(sub, cfg), cfg)
        for axis, arr in enumerate((fl.fx, fl.fy, fl.fz)):
            expect = euler_flux(rho, v, p, E, axis)
            for comp in range(5):
                assert np.allclose(arr[comp], expect[comp], rtol=1e-13, atol=1e-15), (axis, comp)

    def test_mirrored_states_zero_mass_flux(self):
        sub = uniform_subgrid(rho=1.0, v=(0.0, 0.0, 0.0), p=1.0)
        vx = np.zeros((EXT, EXT, EXT))
        for xe in range(EXT):
            vx[:, :, xe] = 0.3 if xe < 6 else -0.3
        sub.fields["sx"][...] = vx
        sub.fields["E"][...] = 1.0 / (GAMMA - 1.0) + 0.5 * vx ** 2
        cfg = HydroConfig()
        fl = flux(sub, reconstruct(sub, cfg), cfg)
        assert np.all(fl.fx[0][:, :, 4] == 0.0)

    def test_max_speed(self):
        sub = uniform_subgrid(rho=1.0, v=(0.5, 0.0, 0.0), p=1.0)
        cfg = HydroConfig()
        fl = flux(sub, reconstruct(sub, cfg), cfg)
        assert abs(fl.max_speed - (0.5 + np.sqrt(GAMMA))) < 1e-14

    def test_nonpositive_density_error_names_cell(self):
        sub = uniform_subgrid()
        cfg = HydroConfig()
        q = reconstruct(sub, cfg)
        q.values[0, :, 4, 4, 4] = -1.0
        with pytest.raises(KernelError, match=r"density.*\(x=.*y=.*z=.*leaf"):
            flux(sub, q, cfg)

    def test_nonpositive_pressure_error(self):
        sub = uniform_subgrid()
        cfg = HydroConfig()
        q = reconstruct(sub, cfg)
        q.values[4, :, 4, 4, 4] = 1e-9
        q.values[1, :, 4, 4, 4] = 1.0
        with pytest.raises(KernelError, match="pressure"):
            flux(sub, q, cfg)

    @pytest.mark.parametrize("backend", BACKENDS[1:])
    def test_backend_matches_scalar_bitwise(self, backend):
        sub = random_hydro_subgrid(np.random.default_rng(33))
        cfg = HydroConfig()
        q = reconstruct(sub, cfg)
        ref = flux(sub, q, cfg, "scalar")
        got = flux(sub, q, cfg, backend)
        assert got.max_speed == ref.max_speed
        for a, b in ((got.fx, ref.fx), (got.fy, ref.fy), (got.fz, ref.fz)):
            assert np.array_equal(bits(a), bits(b))


def zero_fluxes():
    return FluxField(np.zeros((5, 8, 8, 9)), np.zeros((5, 8, 9, 8)), np.zeros((5, 9, 8, 8)), 1.0)


class TestHydroUpdate:
    def test_zero_fluxes_identity(self):
        sub = uniform_subgrid(rho=1.2, v=(0.1, 0.2, 0.3), p=2.0)
        before = {n: sub.interior(n).copy() for n in HYDRO_FIELDS}
        hydro_update(sub, zero_fluxes(), 1e-4, HydroConfig())
        for n in HYDRO_FIELDS:
            assert np.array_equal(sub.interior(n), before[n])

    def test_uniform_state_unchanged(self):
        sub = uniform_subgrid(rho=1.5, v=(0.2, -0.1, 0.05), p=1.1)
        cfg = HydroConfig()
        before = {n: sub.interior(n).copy() for n in HYDRO_FIELDS}
        fl = flux(sub, reconstruct(sub, cfg), cfg)
        hydro_update(sub, fl, cfg.cfl * sub.dx / (3.0 * fl.max_speed), cfg)
        for n in HYDRO_FIELDS:
            assert np.array_equal(sub.interior(n), before[n])

    def test_cfl_violation_rejected(self):
        sub = uniform_subgrid()
        cfg = HydroConfig()
        fl = flux(sub, reconstruct(sub, cfg), cfg)
        with pytest.raises(KernelError, match="CFL"):
            hydro_update(sub, fl, 2.0 * cfg.cfl * sub.dx / fl.max_speed, cfg)

    def test_nonpositive_dt_rejected(self):
        with pytest.raises(KernelError, match="dt"):
            hydro_update(uniform_subgrid(), zero_fluxes(), 0.0, HydroConfig())

    def test_nonpositive_density_after_update_names_cell(self):
        sub = uniform_subgrid()
        fl = zero_fluxes()
        fl.fx[0, 2, 3, 5] = 1e6  # x-face 5 is the right face of cell x=4: drains it
        with pytest.raises(KernelError, match=r"rho after update at interior cell \(x=4, y=3, z=2\)"):
            hydro_update(sub, fl, 1e-3, HydroConfig())

    def test_periodic_pulse_conserves_mass(self):
        def init(X, Y, Z, dx):
            rho = 1.0 + 0.2 * np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2) / 0.02)
            p = np.ones_like(X)
            return {"rho": rho, "sx": rho * 0.1, "sy": np.zeros_like(X), "sz": np.zeros_like(X),
                    "E": p / (GAMMA - 1.0) + 0.5 * rho * 0.01}

        tree = build_unigrid(1, init)
        cfg = HydroConfig()

        def totals():
            dx3 = tree.dx ** 3
            return {n: float(sum(lf.interior(n).sum() for lf in tree.leaves)) * dx3 for n in HYDRO_FIELDS}

        before = totals()
        for _ in range(10):
            s_pre = max(max_wavespeed(leaf, cfg) for leaf in tree.leaves)
            dt = cfg.cfl * tree.dx / (3.0 * s_pre)
            exchange_ghosts(tree, "hydro")
            qs = [reconstruct(leaf, cfg, "emulated8") for leaf in tree.leaves]
            fls = [flux(leaf, q, cfg, "emulated8") for leaf, q in zip(tree.leaves, qs)]
            for leaf, fl in zip(tree.leaves, fls):
                hydro_update(leaf, fl, dt, cfg)
        after = totals()
        assert abs(after["rho"] - before["rho"]) / abs(before["rho"]) <= 1e-12
        assert abs(after["E"] - before["E"]) / abs(before["E"]) <= 1e-12


class TestStencilCoverage:
    """NaN-poisoned ghost cells the stencil must exclude stay excluded
    (reference test_hydro_kernels.py:243-295)."""

    def _run_pipeline(self, sub):
        cfg = HydroConfig()
        q = reconstruct(sub, cfg, "emulated4")
        fl = flux(sub, q, cfg, "emulated4")
        out = np.empty((5, 8, 8, 8))
        for v, name in enumerate(HYDRO_FIELDS):
            net = ((fl.fx[v, :, :, 1:] - fl.fx[v, :, :, :-1]) + (fl.fy[v, :, 1:, :] - fl.fy[v, :, :-1, :])
                   + (fl.fz[v, 1:, :, :] - fl.fz[v, :-1, :, :]))
            out[v] = sub.interior(name) - 1e-3 * net
        return out

    def test_corner_blocks_are_excluded(self):
        sub = random_hydro_subgrid(np.random.default_rng(5))
        for name in HYDRO_FIELDS:
            arr = sub.fields[name]
            for zs in (slice(0, 2), slice(EXT - 2, EXT)):
                for ys in (slice(0, 2), slice(EXT - 2, EXT)):
                    for xs in (slice(0, 2), slice(EXT - 2, EXT)):
                        arr[zs, ys, xs] = np.nan
        assert np.all(np.isfinite(self._run_pipeline(sub)))

    def test_second_ring_edges_are_excluded(self):
        sub = random_hydro_subgrid(np.random.default_rng(6))
        for name in HYDRO_FIELDS:
            arr = sub.fields[name]
            arr[0, 0, :] = np.nan
            arr[0, :, EXT - 1] = np.nan
            arr[EXT - 1, EXT - 1, :] = np.nan
        assert np.all(np.isfinite(self._run_pipeline(sub)))

    def test_face_ghost_poison_reaches_interior(self):
        sub = random_hydro_subgrid(np.random.default_rng(7))
        sub.fields["rho"][6, 6, 1] = np.nan
        assert np.isnan(self._run_pipeline(sub)).any()

"""Host-side logic, CPU only: configs, backend registry, octree data
contract (reference pkg/tests/test_octree.py), slab partition, status-word
decoding, and the slab halo exchange on CPU tensors."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2210_06439_b200 import kernels as K
from paper_2210_06439_b200 import simd
from paper_2210_06439_b200.octree import (DIRECTIONS, EXT, GHOST, N, build_unigrid, exchange_ghosts,
                                          global_field, leaf_iter, neighborhood27, set_global_field,
                                          source_cube)
from paper_2210_06439_b200.slab import Slab, exchange_z_halo_local


class TestConfigs:
    def test_defaults(self):
        h = K.HydroConfig()
        assert h.gamma == 1.4 and h.cfl == 0.4 and h.positivity_floor == 1e-12
        g = K.GravityConfig()
        assert g.theta == 0.34 and g.eps == 0.5 and g.expansion_order == 0

    def test_validation(self):
        for kw in ({"gamma": 1.0}, {"cfl": 1.0}, {"cfl": 0.0}, {"positivity_floor": 0.0}):
            with pytest.raises(ValueError):
                K.HydroConfig(**kw)
        for kw in ({"theta": 0.0}, {"theta": 1.5}, {"eps": 0.0}, {"expansion_order": 2}):
            with pytest.raises(ValueError):
                K.GravityConfig(**kw)

    def test_halo(self):
        assert [K.gravity_halo(t) for t in (1.0, 0.5, 0.34, 0.2, 0.05)] == [1, 2, 2, 5, 8]

    def test_gravity_params_match_reference_expression(self):
        dx = 1.0 / 64
        rad2, eps2 = K.gravity_params(dx, K.GravityConfig())
        rad = dx / 0.34
        assert rad2 == rad * rad and eps2 == (0.5 * dx) * (0.5 * dx)


class TestBackends:
    def test_registry(self):
        assert simd.available_backends() == ("scalar", "emulated2", "emulated4", "emulated8", "emulated16")
        assert simd.get_backend("emulated8").width == 8

    def test_unknown(self):
        with pytest.raises(simd.BackendUnavailableError, match="emulated4"):
            simd.get_backend("avx747")

    def test_native_not_built(self):
        with pytest.raises(simd.BackendUnavailableError, match="native"):
            simd.get_backend("native")

    def test_backend_checked_before_device_work(self):
        tree = build_unigrid(0)
        with pytest.raises(simd.BackendUnavailableError):
            K.reconstruct(tree.leaves[0], K.HydroConfig(), "avx747")


def _linear_fill(tree, name="rho"):
    n = tree.leaves_per_axis * N
    for leaf in tree.leaves:
        cx, cy, cz = leaf.coord
        idx = np.arange(N)
        Z, Y, X = np.meshgrid(cz * N + idx, cy * N + idx, cx * N + idx, indexing="ij")
        leaf.interior(name)[...] = X + 1000.0 * Y + 1000000.0 * Z
    return n


class TestOctree:
    def test_leaf_counts_and_dx(self):
        for L in range(4):
            tree = build_unigrid(L)
            assert len(tree) == 8 ** L and tree.dx == 1.0 / (8 * 2 ** L)

    def test_level_bounds(self):
        with pytest.raises(ValueError):
            build_unigrid(6)

    def test_l1_morton_order(self):
        tree = build_unigrid(1)
        assert len(list(leaf_iter(tree))) == 8
        assert [leaf.coord for leaf in tree.leaves] == [
            (0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (0, 0, 1), (1, 0, 1), (0, 1, 1), (1, 1, 1)]

    def test_sentinels(self):
        tree = build_unigrid(1, lambda X, Y, Z, dx: {"rho": X})
        leaf = tree.leaves[0]
        assert np.all(np.isfinite(leaf.interior("rho"))) and np.isnan(leaf.fields["rho"][0, 0, 0])
        assert np.all(leaf.fields["phi"] == 0.0)

    def test_neighbour_symmetry(self):
        tree = build_unigrid(2)
        for i in range(len(tree)):
            for d in range(26):
                assert tree.neighbor(tree.neighbor(i, d), 25 - d) == i
        for d, (dz, dy, dx) in enumerate(DIRECTIONS):
            assert DIRECTIONS[25 - d] == (-dz, -dy, -dx)

    def test_ghosts_match_periodic_index_map(self):
        tree = build_unigrid(1)
        n = _linear_fill(tree)
        exchange_ghosts(tree, "hydro")
        e = np.arange(EXT)
        for leaf in tree.leaves:
            cx, cy, cz = leaf.coord
            gx = (cx * N + e - GHOST) % n
            gy = (cy * N + e - GHOST) % n
            gz = (cz * N + e - GHOST) % n
            want = gx[None, None, :] + 1000.0 * gy[None, :, None] + 1000000.0 * gz[:, None, None]
            assert np.array_equal(leaf.fields["rho"], want)

    def test_exchange_idempotent_and_field_sets(self):
        tree = build_unigrid(1)
        _linear_fill(tree)
        exchange_ghosts(tree, "hydro")
        snap = [leaf.fields["rho"].copy() for leaf in tree.leaves]
        exchange_ghosts(tree, "hydro")
        assert all(np.array_equal(a.fields["rho"], b) for a, b in zip(tree.leaves, snap))
        with pytest.raises(ValueError, match="field set"):
            exchange_ghosts(tree, "everything")
        t0 = build_unigrid(0)
        t0.leaves[0].interior("mass")[...] = 1.0
        t0.leaves[0].interior("rho")[...] = 1.0
        exchange_ghosts(t0, "gravity")
        assert np.all(t0.leaves[0].fields["mass"] == 1.0) and np.isnan(t0.leaves[0].fields["rho"][0, 0, 0])

    @pytest.mark.parametrize("halo", [0, 2, 3, 8])
    def test_source_cube_is_periodic_window(self, halo):
        tree = build_unigrid(1)
        n = _linear_fill(tree, "mass")
        g = global_field(tree, "mass")
        for leaf_id in (0, 5):
            cube = source_cube(neighborhood27(tree, leaf_id), "mass", halo)
            cx, cy, cz = tree.leaves[leaf_id].coord
            r = np.arange(8 + 2 * halo) - halo
            want = g[np.ix_((cz * 8 + r) % n, (cy * 8 + r) % n, (cx * 8 + r) % n)]
            assert np.array_equal(cube, want)
        with pytest.raises(ValueError):
            source_cube(neighborhood27(tree, 0), "mass", 9)

    def test_global_field_roundtrip(self):
        tree = build_unigrid(2)
        a = np.random.default_rng(0).uniform(size=(32, 32, 32))
        set_global_field(tree, "rho", a)
        assert np.array_equal(global_field(tree, "rho"), a)


class TestSlab:
    def test_partition(self):
        s = Slab(4, 3, 8)
        assert (s.n, s.layers, s.nz, s.z0, s.up, s.down) == (128, 2, 16, 48, 4, 2)
        c = s.global_leaf_coords().numpy()
        assert len(c) == 2 * 16 * 16 and c[:, 2].min() == 6 and c[:, 2].max() == 7
        with pytest.raises(ValueError):
            Slab(2, 0, 3)

    @pytest.mark.parametrize("world", [1, 2, 4])
    def test_local_exchange_equals_periodic_pad(self, world):
        level, pad = 2, 8
        n = 8 << level
        g = torch.from_numpy(np.random.default_rng(1).uniform(size=(2, n, n, n)))
        want = np.pad(g.numpy(), ((0, 0), (pad, pad), (pad, pad), (pad, pad)), mode="wrap")
        nz = n // world
        fields = []
        for r in range(world):
            f = torch.zeros((2, nz + 2 * pad, n + 2 * pad, n + 2 * pad), dtype=torch.float64)
            # interior planes + x/y periodic pads (the device fill's job)
            f[:, pad:pad + nz] = torch.from_numpy(want[:, pad + r * nz:pad + (r + 1) * nz])
            fields.append(f)
        exchange_z_halo_local(fields, pad, nz)
        for r, f in enumerate(fields):
            assert np.array_equal(f.numpy(), want[:, r * nz:r * nz + nz + 2 * pad])


class TestStatusWords:
    def test_flux_error_decoding(self):
        assert K.decode_flux_error(0xFFFFFFFF) == (0, -1)
        key = 12345
        assert K.decode_flux_error((key << 12) | (2 << 10) | 987) == (2, 987)


def test_stacked_hydro_block_is_shared_until_a_field_is_replaced():
    """SubGrid.allocate keeps the hydro fields as views of one (5, 12, 12, 12)
    block, which the drop-in calls pass to the library without a copy; a
    replaced field array falls back to a stacked copy with the same values."""
    leaf = build_unigrid(1).leaves[3]
    rng = np.random.default_rng(0)
    for name in K.HYDRO_FIELDS:
        leaf.fields[name][...] = rng.uniform(size=(EXT, EXT, EXT))
    want = np.stack([leaf.fields[n] for n in K.HYDRO_FIELDS])
    blk = K._stack_hydro(leaf)
    assert blk is leaf.hydro_block and np.array_equal(blk, want)
    leaf.fields["sy"] = leaf.fields["sy"].copy()
    leaf.fields["sy"][0, 0, 0] = -1.0
    want[2, 0, 0, 0] = -1.0
    U = K._stack_hydro(leaf)
    assert U is not leaf.hydro_block and np.array_equal(U, want)


def test_source_cube_is_periodic_window_of_global_field():
    """octree.source_cube (reference octree.py:186-214) == the periodic
    (8+2h)^3 window of the global field around the leaf, every halo 0..8."""
    import numpy as np

    from paper_2210_06439_b200 import octree

    tree = octree.build_unigrid(2)
    rng = np.random.default_rng(5)
    F = rng.random((32, 32, 32))
    octree.set_global_field(tree, "mass", F)
    for lid in (0, 9, 63):
        cx, cy, cz = tree.leaves[lid].coord
        nb = octree.neighborhood27(tree, lid)
        for h in range(0, 9):
            r = np.arange(-h, 8 + h)
            want = F[np.ix_((cz * 8 + r) % 32, (cy * 8 + r) % 32, (cx * 8 + r) % 32)]
            assert np.array_equal(octree.source_cube(nb, "mass", h), want), (lid, h)
    import pytest
    with pytest.raises(ValueError):
        octree.source_cube(nb, "mass", 9)


def test_bench_roofline_traffic_reads_the_m2l_section():
    """bench.py's roofline `traffic` comes from the exact-M2L section of the
    newest committed ncu summary (the file may also hold a P2P capture)."""
    import sys

    from conftest import REPO
    sys.path.insert(0, str(REPO))
    import bench

    traffic, name = bench.m2l_traffic_from_profile()
    assert name is not None and name.endswith("_m2l_L4_ncu_full.txt")
    text = (REPO / "profiles" / name).read_text()
    sect = [t for t in text.split("== ncu --set full")[1:]
            if "m2l_kernel" in t.split("\n", 3)[1] or "m2l_pair_kernel" in t.split("\n", 3)[1]]
    assert sect, name
    assert 1e7 < traffic < 1e9


def test_bench_line_is_strict_json():
    """bench.py prints strict JSON: non-finite floats become null."""
    import json
    import math
    import sys

    from conftest import REPO
    sys.path.insert(0, str(REPO))
    import bench

    line = {"value": float("nan"), "roofline": {"traffic": float("inf"), "frac": 0.5}, "xs": [1.0, -math.inf]}
    out = json.dumps(bench._strict_json(line), allow_nan=False)
    assert json.loads(out) == {"value": None, "roofline": {"traffic": None, "frac": 0.5}, "xs": [1.0, None]}

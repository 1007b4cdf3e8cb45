"""Harness logic without a GPU: scenario configs and initial conditions
(reference pkg/tests/test_scenarios.py:24-93), CSV schema and rows."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import digest
from paper_2210_06439_b200 import driver as D
from paper_2210_06439_b200.octree import global_field


class TestScenarioConfig:
    def test_defaults(self):
        cfg = D.ScenarioConfig("rotating-star-proxy")
        assert cfg.max_level == 3 and cfg.stop_step == 10 and cfg.theta == 0.34
        assert cfg.gravity_per_step == 6 and cfg.hydro_per_step == 3
        assert cfg.gravity.expansion_order == 1 and cfg.gravity.eps == 0.5

    def test_blast_runs_zero_gravity(self):
        assert D.ScenarioConfig("blast").gravity_per_step == 0

    def test_validation(self):
        with pytest.raises(ValueError, match="scenario"):
            D.ScenarioConfig("supernova")
        with pytest.raises(ValueError, match="stop_step"):
            D.ScenarioConfig("blast", stop_step=0)
        with pytest.raises(ValueError):
            D.ScenarioConfig("blast", max_level=6)


class TestInitScenario:
    @pytest.mark.parametrize("level", [0, 1, 2])
    def test_blast_total_energy(self, level):
        tree = D.init_scenario(D.ScenarioConfig("blast", max_level=level, stop_step=1))
        dx3 = tree.dx ** 3
        n_cells = 512 * 8 ** level
        expect = D.BLAST_BACKGROUND_E * (n_cells - 8) * dx3 + D.BLAST_CENTER_E * 8 * dx3
        got = float(sum(leaf.interior("E").sum() for leaf in tree.leaves)) * dx3
        assert abs(got - expect) <= 1e-15 * abs(expect)

    def test_blast_center_block(self):
        tree = D.init_scenario(D.ScenarioConfig("blast", max_level=1, stop_step=1))
        E = global_field(tree, "E")
        hot = {tuple(h) for h in np.argwhere(E == D.BLAST_CENTER_E)}
        n = E.shape[0]
        m = (n // 2 - 1, n // 2)
        assert hot == {(a, b, c) for a in m for b in m for c in m}

    def test_star_rotation_and_masses(self):
        tree = D.init_scenario(D.ScenarioConfig("rotating-star-proxy", max_level=1, stop_step=1))
        leaf = tree.leaves[0]
        X, Y, Z = leaf.cell_centers()
        assert np.allclose(leaf.interior("sx") / leaf.interior("rho"), -(Y - 0.5), rtol=1e-13, atol=1e-15)
        assert np.allclose(leaf.interior("sy") / leaf.interior("rho"), X - 0.5, rtol=1e-13, atol=1e-15)
        assert np.all(leaf.interior("sz") == 0.0)
        leaf = tree.leaves[3]
        assert np.array_equal(leaf.interior("mass"), leaf.interior("rho") * leaf.dx ** 3)

    @pytest.mark.parametrize("key", ["rotating-star-proxy_L1_s2", "blast_L1_s3", "rotating-star-proxy_L2_s1"])
    def test_initial_state_matches_reference_bits(self, manifest, key):
        rec = manifest["scenarios"][key]
        name = key.rsplit("_L", 1)[0]
        tree = D.init_scenario(D.ScenarioConfig(name, max_level=rec["level"], stop_step=1))
        for f, d in rec["input_digests"].items():
            if digest(global_field(tree, f)) != d:
                pytest.fail("input generator mismatch: numpy transcendental loops differ on this host -- the golden inputs cannot be reproduced, parity coverage would be lost")


class TestCsv:
    def _result(self):
        cfg = D.ScenarioConfig("blast", max_level=0, stop_step=1)
        recs = (D.ProfileRecord("reconstruct", 3, 300), D.ProfileRecord("flux", 3, 600),
                D.ProfileRecord("hydro_update", 3, 90), D.ProfileRecord("total", 1, 5000))
        return D.RunResult(cfg, "scalar", 1, 1, None, recs, 5e-6, D.LaunchStats())

    def test_header_layout(self):
        assert D.CSV_HEADER.split(",") == ["scenario", "backend", "simd_width", "threads", "tasks_per_multipole",
                                           "kernel", "count", "mean_ns", "total_ns", "computation_s"]

    def test_expected_row_count(self):
        assert D.expected_row_count("rotating-star-proxy", 6) == 36
        assert D.expected_row_count("blast", 6) == 24

    def test_bench_records_order_and_write(self, tmp_path):
        rows = D.bench_records(self._result())
        assert [r.kernel for r in rows] == ["reconstruct", "flux", "hydro_update", "total"]
        assert rows[0].mean_ns == 100.0 and rows[-1].computation_s == 5e-6
        path = tmp_path / "bench.csv"
        D.write_csv(str(path), rows)
        D.write_csv(str(path), rows)
        raw = path.read_bytes().decode("utf-8")
        lines = [ln for ln in raw.split("\n") if ln]
        assert lines[0] == D.CSV_HEADER and "\r" not in raw and len(lines) == 1 + 2 * 4
        assert lines[1] == "blast,cuda,32,1,1,reconstruct,3,100.0,300,5e-06"

    def test_argument_validation(self):
        cfg = D.ScenarioConfig("blast", max_level=0, stop_step=1)
        from paper_2210_06439_b200.simd import BackendUnavailableError
        with pytest.raises(BackendUnavailableError):
            D.run_scenario(cfg, backend="sse9")
        with pytest.raises(ValueError, match="tasks_per_multipole"):
            D.run_scenario(cfg, tasks_per_multipole=0)
        with pytest.raises(ValueError, match="hydro_kernel"):
            D.run_scenario(cfg, hydro_kernel="turbo")
        with pytest.raises(ValueError):
            D.sweep(cfg, [], ["scalar"], "x.csv")

"""The plotting frontend (plots.py; the reference's frontend/ figure math and
CLI behaviour) on harness CSVs written by driver.write_csv."""

from __future__ import annotations

import xml.etree.ElementTree as ET

import pytest

from paper_2210_06439_b200 import plots
from paper_2210_06439_b200.driver import CSV_HEADER, BenchRecord, write_csv

KERNELS = ("reconstruct", "flux", "hydro_update", "monopole", "multipole", "total")


def _rows(scenario="rotating-star-proxy", backends=("scalar", "emulated8", "cuda"), threads=(1, 2, 4)):
    # mean_ns: scalar 1000*(k+1), emulated8 4x faster, cuda 50x; total computation scales 1/p^0.9
    speed = {"scalar": 1.0, "emulated8": 4.0, "cuda": 50.0}
    out = []
    for p in threads:
        for b in backends:
            comp = 10.0 / speed[b] / p ** 0.9
            for k, kern in enumerate(KERNELS):
                mean = 1000.0 * (k + 1) / speed[b] / (p if kern == "total" else 1)
                out.append(BenchRecord(scenario, b, 8, p, 1, kern, 4, mean, int(4 * mean), comp))
    return out


def test_figure_math(tmp_path):
    csv = tmp_path / "sweep.csv"
    write_csv(str(csv), _rows())
    rows = plots.load_rows(str(csv))
    sp = {(k, b): v for k, b, v in plots.speedups(rows)}
    assert sp[("flux", "emulated8")] == pytest.approx(4.0)
    assert sp[("multipole", "cuda")] == pytest.approx(50.0)
    assert sp[("reconstruct", "scalar")] == 1.0
    assert [k for k, b, _ in plots.speedups(rows) if b == "cuda"] == list(KERNELS)  # harness order
    sc = plots.scaling(rows)
    eff = {(b, p): e for b, p, _, e in sc}
    assert eff[("scalar", 1)] == pytest.approx(1.0)
    assert eff[("emulated8", 4)] == pytest.approx(1.0 / (4 * 4 ** -0.9))
    legacy = [r for r in _rows(scenario="blast", backends=("scalar",))]
    legacy = [BenchRecord(r.scenario, "legacy", 8, r.threads, 1, r.kernel, r.count, r.mean_ns * 1.5, r.total_ns,
                          r.computation_s * 1.5) for r in legacy]
    blast = _rows(scenario="blast")
    hc = plots.hydro_compare(plots.parse_csv(_text(blast), "b"), plots.parse_csv(_text(legacy), "l"), "cuda")
    d = {(g, v): c for g, v, c in hc}
    assert d[("one core", "legacy")] == pytest.approx(15.0)
    assert d[("all cores", "simd")] == pytest.approx(10.0 / 50 / 4 ** 0.9)


def _text(records) -> str:
    return CSV_HEADER + "\n" + "\n".join(r.csv_row() for r in records) + "\n"


def test_cli_writes_three_svgs(tmp_path):
    csv, leg = tmp_path / "sweep.csv", tmp_path / "legacy.csv"
    write_csv(str(csv), _rows() + _rows(scenario="blast"))
    legacy = [BenchRecord("blast", "legacy", 8, r.threads, 1, r.kernel, r.count, r.mean_ns, r.total_ns,
                          r.computation_s * 2) for r in _rows(scenario="blast", backends=("scalar",))]
    write_csv(str(leg), legacy)
    out = tmp_path / "fig"
    assert plots.main(["--filename", str(csv), "--simd-key", "cuda", "--outdir", str(out),
                       "--legacy-files", str(leg)]) == 0
    names = sorted(p.name for p in out.iterdir())
    assert names == ["hydro_compare.svg", "node_scaling.svg", "simd_speedup.svg"]
    ns = {"s": "http://www.w3.org/2000/svg"}
    sp = ET.parse(out / "simd_speedup.svg").getroot()
    bars = sp.findall(".//s:rect[@class='bar']", ns)
    assert len(bars) == 2 * len(KERNELS)           # emulated8 + cuda per kernel (scalar omitted)
    hl = [b for b in bars if b.get("stroke") == "black"]
    assert {b.get("data-label") for b in hl} == {"cuda"}
    sc = ET.parse(out / "node_scaling.svg").getroot()
    assert len(sc.findall(".//s:polyline", ns)) == 2 * 3  # two panels x three backends
    hc = ET.parse(out / "hydro_compare.svg").getroot()
    assert len(hc.findall(".//s:rect[@class='bar']", ns)) == 6
    # identical input -> identical figures
    out2 = tmp_path / "fig2"
    plots.main(["--filename", str(csv), "--simd-key", "cuda", "--outdir", str(out2), "--legacy-files", str(leg)])
    assert (out / "simd_speedup.svg").read_text() == (out2 / "simd_speedup.svg").read_text()


def test_errors(tmp_path, capsys):
    with pytest.raises(ValueError, match="header does not match"):
        plots.parse_csv("a,b\n1,2\n", "x.csv")
    with pytest.raises(ValueError, match="empty file"):
        plots.parse_csv("\n", "x.csv")
    bad = CSV_HEADER + "\ns,scalar,8,1,1,flux,1,nan,1,1.0\n"
    with pytest.raises(ValueError, match=r"x.csv:2: mean_ns is not a finite number"):
        plots.parse_csv(bad, "x.csv")
    with pytest.raises(ValueError, match="expected 10 fields"):
        plots.parse_csv(CSV_HEADER + "\n1,2\n", "x.csv")
    rows = plots.parse_csv(_text(_rows(backends=("emulated8",))), "y")
    with pytest.raises(ValueError, match="missing scalar baseline at threads=1 for kernel 'reconstruct'"):
        plots.speedups(rows)
    with pytest.raises(ValueError, match="simd key 'avx' not present"):
        plots.require_simd_key(rows, "avx")
    with pytest.raises(ValueError, match="at least two thread counts"):
        plots.scaling(plots.parse_csv(_text(_rows(threads=(1,))), "z"))
    with pytest.raises(ValueError, match="missing hydro variant"):
        plots.hydro_compare(rows, rows, "cuda")
    csv = tmp_path / "s.csv"
    write_csv(str(csv), _rows())
    assert plots.main(["--filename", str(csv), "--simd-key", "cuda", "--outdir", str(tmp_path / "o")]) == 0
    assert "hydro comparison skipped" in capsys.readouterr().err
    assert plots.main(["--filename", str(tmp_path / "nope.csv"), "--simd-key", "cuda"]) == 1

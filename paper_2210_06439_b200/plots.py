"""Plotting frontend for the benchmark CSV (the reference's TypeScript
`frontend/` -- cli.ts, csv.ts, figures.ts, svg.ts -- rebuilt in Python
because node is not available here).

Reads the harness CSV written by ``driver.write_csv`` (the reference's schema,
driver.py:41-68 / 233-240, consumed verbatim) and writes the same three SVG
figures:

* ``simd_speedup.svg``  per-kernel single-thread speedup of every backend over
  ``scalar`` (the ``--simd-key`` backend outlined);
* ``node_scaling.svg``  ``total`` computation time vs thread count per
  backend, with a parallel-efficiency panel T(1) / (p T(p));
* ``hydro_compare.svg`` one-core / all-cores computation of the ``legacy``,
  ``scalar`` and simd hydro variants (legacy rows from ``--legacy-files``;
  the scenario found there selects the rows compared).

Usage::

    python -m paper_2210_06439_b200.plots --filename sweep.csv --simd-key emulated8 \
        --outdir figures [--legacy-files legacy.csv ...]

The figure numbers are pure functions of the rows (``speedups``,
``scaling``, ``hydro_compare``) with fixed sort orders, so identical input
gives identical files.  Errors mirror the reference tool: a header that is
not the harness schema, a non-finite field, a missing ``scalar`` baseline,
an absent ``--simd-key``, fewer than two thread counts, a missing hydro
variant -- each raises ``ValueError`` naming the file / line / what is
missing.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
from dataclasses import dataclass
from xml.sax.saxutils import escape

from .driver import CSV_HEADER, KERNEL_ORDER

__all__ = ["Row", "parse_csv", "load_rows", "speedups", "scaling", "hydro_compare", "bar_chart_svg",
           "line_chart_svg", "plot", "main"]


@dataclass(frozen=True)
class Row:
    scenario: str
    backend: str
    simd_width: float
    threads: float
    tasks_per_multipole: float
    kernel: str
    count: float
    mean_ns: float
    total_ns: float
    computation_s: float


_NUMERIC = ("simd_width", "threads", "tasks_per_multipole", None, "count", "mean_ns", "total_ns", "computation_s")


def parse_csv(text: str, source: str = "<csv>") -> list[Row]:
    """Rows of one harness CSV (fixed schema, no quoting, blank lines ignored)."""
    lines = [ln for ln in text.split("\n") if ln.strip()]
    if not lines:
        raise ValueError(f"{source}: empty file")
    if lines[0] != CSV_HEADER:
        raise ValueError(f"{source}: header does not match the harness schema\n"
                         f"  got:      {lines[0]}\n  expected: {CSV_HEADER}")
    rows = []
    for n, line in enumerate(lines[1:], start=2):
        f = line.split(",")
        if len(f) != 10:
            raise ValueError(f"{source}:{n}: expected 10 fields, got {len(f)}")
        vals = []
        for name, text_v in zip(_NUMERIC, f[2:]):
            if name is None:  # the kernel column
                vals.append(text_v)
                continue
            try:
                v = float(text_v)
            except ValueError:
                v = math.nan
            if not math.isfinite(v):
                raise ValueError(f"{source}:{n}: {name} is not a finite number: {text_v}")
            vals.append(v)
        rows.append(Row(f[0], f[1], vals[0], vals[1], vals[2], vals[3], vals[4], vals[5], vals[6], vals[7]))
    return rows


def load_rows(path: str) -> list[Row]:
    if not os.path.exists(path):
        raise ValueError(f"no such file: {path}")
    with open(path, encoding="utf-8") as fh:
        return parse_csv(fh.read(), path)


def _kernel_key(k: str):
    return (KERNEL_ORDER.index(k) if k in KERNEL_ORDER else len(KERNEL_ORDER), k)


def _mean(xs) -> float:
    xs = list(xs)
    return sum(xs) / len(xs)


def require_simd_key(rows: list[Row], simd_key: str) -> None:
    if not any(r.backend == simd_key for r in rows):
        present = ", ".join(sorted({r.backend for r in rows}))
        raise ValueError(f"simd key '{simd_key}' not present in the data (backends: {present})")


def speedups(rows: list[Row]) -> list[tuple[str, str, float]]:
    """(kernel, backend, scalar mean_ns / backend mean_ns) at threads == 1,
    kernels in the harness order, backends sorted."""
    one = [r for r in rows if r.threads == 1]
    out = []
    for kernel in sorted({r.kernel for r in one}, key=_kernel_key):
        base = [r.mean_ns for r in one if r.kernel == kernel and r.backend == "scalar"]
        if not base:
            raise ValueError(f"missing scalar baseline at threads=1 for kernel '{kernel}'")
        b = _mean(base)
        for backend in sorted({r.backend for r in one}):
            mine = [r.mean_ns for r in one if r.kernel == kernel and r.backend == backend]
            if mine:
                out.append((kernel, backend, b / _mean(mine)))
    return out


def scaling(rows: list[Row]) -> list[tuple[str, float, float, float]]:
    """(backend, threads, mean total computation_s, efficiency T(1)/(p T(p)))."""
    totals = [r for r in rows if r.kernel == "total"]
    counts = sorted({r.threads for r in totals})
    if len(counts) < 2:
        raise ValueError(f"scaling needs at least two thread counts, found {len(counts)} "
                         f"({', '.join(f'{c:g}' for c in counts)})")
    out = []
    for backend in sorted({r.backend for r in totals}):
        mine = [r for r in totals if r.backend == backend]
        t1 = [r.computation_s for r in mine if r.threads == 1]
        if not t1:
            continue
        t1m = _mean(t1)
        for p in counts:
            here = [r.computation_s for r in mine if r.threads == p]
            if here:
                tp = _mean(here)
                out.append((backend, p, tp, t1m / (p * tp)))
    return out


def hydro_compare(rows: list[Row], legacy_rows: list[Row], simd_key: str) -> list[tuple[str, str, float]]:
    """(group 'one core'|'all cores', variant 'legacy'|'scalar'|'simd', mean total computation_s) for
    the scenario(s) the legacy rows were produced with; one core = the fewest threads present."""
    if not legacy_rows:
        raise ValueError("hydro comparison requires legacy rows (see --legacy-files)")
    scen = {r.scenario for r in legacy_rows}
    scoped = [r for r in rows if r.scenario in scen and r.kernel == "total"]
    variants = {"legacy": [r for r in legacy_rows if r.kernel == "total"],
                "scalar": [r for r in scoped if r.backend == "scalar"],
                "simd": [r for r in scoped if r.backend == simd_key]}
    missing = [k for k, v in variants.items() if not v]
    if missing:
        present = [k for k, v in variants.items() if v]
        raise ValueError(f"missing hydro variant(s): {', '.join(missing)} (present: {', '.join(present) or 'none'})")
    out = []
    for variant, vr in variants.items():
        lo, hi = min(r.threads for r in vr), max(r.threads for r in vr)
        out.append(("one core", variant, _mean(r.computation_s for r in vr if r.threads == lo)))
        out.append(("all cores", variant, _mean(r.computation_s for r in vr if r.threads == hi)))
    return out


# -- SVG ---------------------------------------------------------------------

_PALETTE = ["#4e79a7", "#f28e2b", "#59a14f", "#e15759", "#76b7b2", "#edc948", "#b07aa1", "#ff9da7", "#9c755f"]
W, H, ML, MR, MT, MB = 760, 420, 70, 150, 40, 70


def _nice_max(v: float) -> float:
    if v <= 0:
        return 1.0
    e = 10 ** math.floor(math.log10(v))
    for m in (1, 2, 2.5, 5, 10):
        if m * e >= v:
            return m * e
    return 10 * e


def _text(x, y, s, size=12, anchor="middle", weight="normal", rotate=None) -> str:
    rot = f' transform="rotate({rotate} {x:.1f} {y:.1f})"' if rotate is not None else ""
    return (f'<text x="{x:.1f}" y="{y:.1f}" font-size="{size}" text-anchor="{anchor}" '
            f'font-weight="{weight}" font-family="sans-serif"{rot}>{escape(str(s))}</text>')


def _frame(title: str, ylabel: str, ymax: float, x0, y0, w, h, ticks=5) -> list[str]:
    out = [_text(x0 + w / 2, y0 - 14, title, 15, weight="bold"),
           f'<line x1="{x0}" y1="{y0 + h}" x2="{x0 + w}" y2="{y0 + h}" stroke="black"/>',
           f'<line x1="{x0}" y1="{y0}" x2="{x0}" y2="{y0 + h}" stroke="black"/>',
           _text(x0 - 50, y0 + h / 2, ylabel, 12, rotate=-90)]
    for i in range(ticks + 1):
        v = ymax * i / ticks
        y = y0 + h - h * i / ticks
        out.append(f'<line x1="{x0 - 4}" y1="{y:.1f}" x2="{x0 + w}" y2="{y:.1f}" stroke="#ddd"/>')
        out.append(_text(x0 - 8, y + 4, f"{v:g}", 10, anchor="end"))
    return out


def bar_chart_svg(title: str, ylabel: str, groups: list[tuple[str, list[tuple[str, float, bool]]]],
                  ref_line: float | None = None) -> str:
    """Grouped bars: groups = [(group label, [(bar label, value, highlight), ...]), ...]."""
    labels = sorted({b[0] for _, bars in groups for b in bars})
    color = {lab: _PALETTE[i % len(_PALETTE)] for i, lab in enumerate(labels)}
    vmax = _nice_max(max([b[1] for _, bars in groups for b in bars] + [ref_line or 0.0]))
    x0, y0, w, h = ML, MT, W - ML - MR, H - MT - MB
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" viewBox="0 0 {W} {H}">',
           '<rect width="100%" height="100%" fill="white"/>'] + _frame(title, ylabel, vmax, x0, y0, w, h)
    gw = w / max(len(groups), 1)
    for gi, (glabel, bars) in enumerate(groups):
        bw = gw * 0.8 / max(len(bars), 1)
        for bi, (blabel, val, hl) in enumerate(bars):
            bh = h * val / vmax
            x = x0 + gi * gw + gw * 0.1 + bi * bw
            stroke = ' stroke="black" stroke-width="2.5"' if hl else ""
            out.append(f'<rect class="bar" data-group="{escape(glabel)}" data-label="{escape(blabel)}" '
                       f'data-value="{val:.6g}" x="{x:.1f}" y="{y0 + h - bh:.1f}" width="{bw * 0.92:.1f}" '
                       f'height="{bh:.1f}" fill="{color[blabel]}"{stroke}/>')
        out.append(_text(x0 + gi * gw + gw / 2, y0 + h + 18, glabel, 11))
    if ref_line is not None:
        y = y0 + h - h * ref_line / vmax
        out.append(f'<line x1="{x0}" y1="{y:.1f}" x2="{x0 + w}" y2="{y:.1f}" stroke="black" '
                   f'stroke-dasharray="5,4"/>')
    for i, lab in enumerate(labels):
        y = y0 + 10 + 18 * i
        out.append(f'<rect x="{x0 + w + 16}" y="{y - 9}" width="12" height="12" fill="{color[lab]}"/>')
        out.append(_text(x0 + w + 34, y + 1, lab, 11, anchor="start"))
    out.append("</svg>")
    return "\n".join(out) + "\n"


def line_chart_svg(title: str, panels: list[tuple[str, list[tuple[str, list[tuple[float, float]]]]]],
                   xlabel: str) -> str:
    """Side-by-side line panels: panels = [(ylabel, [(series label, [(x, y), ...]), ...]), ...]."""
    labels = sorted({s[0] for _, series in panels for s in series})
    color = {lab: _PALETTE[i % len(_PALETTE)] for i, lab in enumerate(labels)}
    pw = (W - ML - MR) / len(panels)
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" viewBox="0 0 {W} {H}">',
           '<rect width="100%" height="100%" fill="white"/>', _text(W / 2, 18, title, 15, weight="bold")]
    for pi, (ylabel, series) in enumerate(panels):
        xs = [p[0] for _, pts in series for p in pts]
        xmax = max(xs) if xs else 1.0
        ymax = _nice_max(max([p[1] for _, pts in series for p in pts] + [0.0]))
        x0, y0, w, h = ML + pi * pw + (20 if pi else 0), MT + 10, pw - 60, H - MT - MB - 10
        out += _frame("", ylabel, ymax, x0, y0, w, h)
        out.append(_text(x0 + w / 2, y0 + h + 36, xlabel, 12))
        for xv in sorted(set(xs)):
            out.append(_text(x0 + w * xv / xmax, y0 + h + 16, f"{xv:g}", 10))
        for lab, pts in series:
            pts = sorted(pts)
            path = " ".join(f"{x0 + w * x / xmax:.1f},{y0 + h - h * y / ymax:.1f}" for x, y in pts)
            out.append(f'<polyline class="series" data-label="{escape(lab)}" points="{path}" fill="none" '
                       f'stroke="{color[lab]}" stroke-width="2"/>')
            for x, y in pts:
                out.append(f'<circle cx="{x0 + w * x / xmax:.1f}" cy="{y0 + h - h * y / ymax:.1f}" r="3" '
                           f'fill="{color[lab]}"/>')
    for i, lab in enumerate(labels):
        y = MT + 20 + 18 * i
        out.append(f'<rect x="{W - MR + 16}" y="{y - 9}" width="12" height="12" fill="{color[lab]}"/>')
        out.append(_text(W - MR + 34, y + 1, lab, 11, anchor="start"))
    out.append("</svg>")
    return "\n".join(out) + "\n"


# -- CLI ---------------------------------------------------------------------

def plot(filename: str, simd_key: str, outdir: str, legacy_files=()) -> list[str]:
    """Write the figures for one CSV; returns the paths written (the hydro
    comparison is skipped with a notice on stderr without legacy files)."""
    rows = load_rows(filename)
    require_simd_key(rows, simd_key)
    os.makedirs(outdir, exist_ok=True)
    written = []
    sp = [b for b in speedups(rows) if b[1] != "scalar"]
    groups = [(k, [(b, v, b == simd_key) for kk, b, v in sp if kk == k])
              for k in sorted({k for k, _, _ in sp}, key=_kernel_key)]
    p = os.path.join(outdir, "simd_speedup.svg")
    with open(p, "w", encoding="utf-8") as fh:
        fh.write(bar_chart_svg("Single-core SIMD speedup over scalar", "speedup", groups, 1.0))
    written.append(p)
    pts = scaling(rows)
    backends = sorted({b for b, *_ in pts})
    timing = [(b, [(t, c) for bb, t, c, _ in pts if bb == b]) for b in backends]
    eff = [(b, [(t, e) for bb, t, _, e in pts if bb == b]) for b in backends]
    p = os.path.join(outdir, "node_scaling.svg")
    with open(p, "w", encoding="utf-8") as fh:
        fh.write(line_chart_svg("Node-level scaling (total)", [("computation [s]", timing),
                                                                ("parallel efficiency", eff)], "threads"))
    written.append(p)
    if legacy_files:
        legacy = [r for f in legacy_files for r in load_rows(f)]
        bars = hydro_compare(rows, legacy, simd_key)
        groups = [(g, [(v, c, v == "simd") for gg, v, c in bars if gg == g]) for g in ("one core", "all cores")]
        p = os.path.join(outdir, "hydro_compare.svg")
        with open(p, "w", encoding="utf-8") as fh:
            fh.write(bar_chart_svg(f"Hydro implementations ({', '.join(sorted({r.scenario for r in legacy}))})",
                                   "computation [s]", groups))
        written.append(p)
    else:
        print("hydro comparison skipped: no --legacy-files given", file=sys.stderr)
    return written


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2210_06439_b200.plots", description=__doc__.split("\n\n")[0])
    ap.add_argument("--filename", required=True, help="harness CSV (driver.write_csv schema)")
    ap.add_argument("--simd-key", required=True, help="backend highlighted as 'simd'")
    ap.add_argument("--outdir", default="figures")
    ap.add_argument("--legacy-files", nargs="*", default=[], help="CSV(s) from --hydro-kernel legacy runs")
    a = ap.parse_args(argv)
    try:
        for p in plot(a.filename, a.simd_key, a.outdir, a.legacy_files):
            print(p)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())

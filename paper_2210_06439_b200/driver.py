"""Experiment harness on the B200 backend -- the reference driver's API
(reference pkg/src/simdgrid/driver.py:1-276 and scenarios.py:1-113) with the
per-leaf thread-pool jobs replaced by the batched device step.

``run_scenario`` runs the reference timestep (driver.py:163-174) with one
launch per kernel over all leaves, times every kernel with CUDA events, and
returns the reference's ``RunResult``: final tree (bit-identical to the
reference run), per-kernel ``ProfileRecord`` s whose ``count`` is the number
of per-leaf kernel evaluations (so ``mean_ns`` stays "per subgrid", the
quantity the reference CSV and plots use), and the total wall time.
``bench_records`` / ``write_csv`` / ``sweep`` emit the reference CSV schema
unchanged (backend column ``cuda``, simd_width = warp width 32).
"""

from __future__ import annotations

import io
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import simd
from .kernels import GravityConfig, HydroConfig
from .octree import HYDRO_FIELDS, Octree, build_unigrid, global_field, set_global_field

__all__ = ["SCENARIO_NAMES", "ScenarioConfig", "init_scenario", "KERNEL_ORDER", "CSV_HEADER", "ProfileRecord",
           "BenchRecord", "LaunchStats", "RunResult", "run_scenario", "bench_records", "write_csv",
           "expected_row_count", "sweep", "BLAST_BACKGROUND_E", "BLAST_CENTER_E"]

SCENARIO_NAMES = ("rotating-star-proxy", "blast")
BLAST_BACKGROUND_E = 1e-3
BLAST_CENTER_E = 10.0
STAR_PEAK_RHO = 10.0
STAR_SIGMA = 1.0 / 8.0
STAR_OMEGA = 1.0
STAR_K = 1.0
STAR_ATMOSPHERE = 0.05

KERNEL_ORDER = ("reconstruct", "flux", "hydro_update", "monopole", "multipole")
HYDRO_KERNELS = ("cuda", "simd", "scalar", "legacy")  # the first three run the same bit-exact kernels
GRAVITY_KERNELS = ("cuda", "simd", "scalar")
WARP_WIDTH = 32

CSV_HEADER = ("scenario,backend,simd_width,threads,tasks_per_multipole,"
              "kernel,count,mean_ns,total_ns,computation_s")


@dataclass(frozen=True)
class ScenarioConfig:
    """reference scenarios.py:32-62"""
    name: str
    max_level: int = 3
    stop_step: int = 10
    theta: float = 0.34
    expansion_order: int = 1
    disable_output: bool = False
    hydro: HydroConfig = field(default_factory=HydroConfig)

    def __post_init__(self):
        if self.name not in SCENARIO_NAMES:
            raise ValueError(f"unknown scenario {self.name!r}; expected one of {SCENARIO_NAMES}")
        if self.stop_step < 1:
            raise ValueError(f"stop_step must be >= 1, got {self.stop_step}")
        if not 0 <= self.max_level <= 5:
            raise ValueError(f"max_level must be in [0, 5], got {self.max_level}")

    @property
    def gravity_per_step(self) -> int:
        return 6 if self.name == "rotating-star-proxy" else 0

    @property
    def hydro_per_step(self) -> int:
        return 3

    @property
    def gravity(self) -> GravityConfig:
        return GravityConfig(theta=self.theta, expansion_order=self.expansion_order)


def _blast_init(gamma: float):
    def init(X, Y, Z, dx):
        rho = np.ones_like(X)
        E = np.full_like(X, BLAST_BACKGROUND_E)
        center = (np.abs(X - 0.5) < dx) & (np.abs(Y - 0.5) < dx) & (np.abs(Z - 0.5) < dx)
        E[center] = BLAST_CENTER_E
        zero = np.zeros_like(X)
        return {"rho": rho, "sx": zero, "sy": zero.copy(), "sz": zero.copy(), "E": E, "mass": rho * dx**3}

    return init


def _rotating_star_init(gamma: float):
    def init(X, Y, Z, dx):
        r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - 0.5) ** 2
        rho = np.maximum(STAR_PEAK_RHO * np.exp(-r2 / (2.0 * STAR_SIGMA**2)), STAR_ATMOSPHERE)
        vx = -STAR_OMEGA * (Y - 0.5)
        vy = STAR_OMEGA * (X - 0.5)
        p = STAR_K * rho**gamma
        E = p / (gamma - 1.0) + 0.5 * rho * (vx**2 + vy**2)
        return {"rho": rho, "sx": rho * vx, "sy": rho * vy, "sz": np.zeros_like(X), "E": E, "mass": rho * dx**3}

    return init


def init_scenario(cfg: ScenarioConfig) -> Octree:
    """Initial interior state (reference scenarios.py:65-113); the same numpy
    expressions evaluated leaf by leaf, so the bits match the reference's."""
    gamma = cfg.hydro.gamma
    if cfg.name == "blast":
        return build_unigrid(cfg.max_level, _blast_init(gamma))
    return build_unigrid(cfg.max_level, _rotating_star_init(gamma))


@dataclass(frozen=True)
class ProfileRecord:
    name: str
    count: int
    total_ns: int

    @property
    def mean_ns(self) -> float:
        return self.total_ns / self.count


@dataclass(frozen=True)
class BenchRecord:
    scenario: str
    backend: str
    simd_width: int
    threads: int
    tasks_per_multipole: int
    kernel: str
    count: int
    mean_ns: float
    total_ns: int
    computation_s: float

    def csv_row(self) -> str:
        return (f"{self.scenario},{self.backend},{self.simd_width},{self.threads},"
                f"{self.tasks_per_multipole},{self.kernel},{self.count},"
                f"{self.mean_ns!r},{self.total_ns},{self.computation_s!r}")


@dataclass
class LaunchStats:
    """The reference counts pool tasks (runtime.py:160-165); here every kernel
    is one device launch over all leaves."""
    spawned: int = 0
    inlined: int = 0
    gpu_launches: int = 0


@dataclass
class RunResult:
    config: ScenarioConfig
    backend: str
    threads: int
    tasks_per_multipole: int
    tree: Octree
    records: tuple
    computation_s: float
    launch_stats: LaunchStats


# device kernels -> the reference's timed kernel names (driver.py:127-160);
# cluster aggregation belongs to multipole_prepare, which the reference does
# not time, so it only shows in "total"
_TIMER_TO_KERNEL = {"p2p": "monopole", "m2l": "multipole", "reconstruct": "reconstruct", "flux": "flux",
                    "hydro_update": "hydro_update"}


def run_scenario(cfg: ScenarioConfig, backend: str = "scalar", threads: int = 1, tasks_per_multipole: int = 1,
                 hydro_kernel: str = "cuda", gravity_kernel: str = "cuda", profiler=None) -> RunResult:
    """Execute ``cfg.stop_step`` timesteps on the GPU (reference driver.py:91-189)."""
    import torch

    from . import _lib
    from .grid import UnigridState

    bk = simd.get_backend(backend)
    if tasks_per_multipole < 1:
        raise ValueError(f"tasks_per_multipole must be >= 1, got {tasks_per_multipole}")
    if hydro_kernel not in HYDRO_KERNELS:
        raise ValueError(f"hydro_kernel must be one of {HYDRO_KERNELS}, got {hydro_kernel!r}")
    if gravity_kernel not in GRAVITY_KERNELS:
        raise ValueError(f"gravity_kernel must be one of {GRAVITY_KERNELS}, got {gravity_kernel!r}")

    tree = init_scenario(cfg)
    # per-kernel records in the reference's per-leaf semantics: the unfused
    # reconstruct -> flux pair keeps "reconstruct" and "flux" separate
    st = UnigridState(cfg.max_level, cfg.hydro, cfg.gravity, fused_hydro=False,
                      legacy_flux=hydro_kernel == "legacy")
    st.load({name: global_field(tree, name) for name in HYDRO_FIELDS})
    st.timers = {}
    st.overlap_p2p = False  # every kernel timed on its own, as the reference's profile
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    t0 = time.perf_counter_ns()
    for step in range(cfg.stop_step):
        if cfg.gravity_per_step:
            st.set_mass()
            for _ in range(cfg.gravity_per_step):
                st.gravity_iteration()
        st.wavespeed_dt()
        for _ in range(cfg.hydro_per_step):
            st.hydro_iteration()
            st.check_errors(step)  # the reference raises "step N: ..." at the failing job
    torch.cuda.synchronize()
    total_ns = time.perf_counter_ns() - t0

    recs = {}
    for timer, evs in st.timers.items():
        name = _TIMER_TO_KERNEL.get(timer)
        if name is None:
            continue
        ns = int(round(sum(a.elapsed_time(b) for a, b in evs) * 1e6))
        c, t = recs.get(name, (0, 0))
        recs[name] = (c + len(evs) * st.nleaves, t + ns)
    records = tuple(ProfileRecord(n, c, t) for n, (c, t) in recs.items()) + (ProfileRecord("total", 1, total_ns),)
    if profiler is not None:
        # a profiling.CudaProfiler (or anything with add(name, count, total_ns))
        for r in records:
            profiler.add(r.name, r.count, r.total_ns)

    out = st.fetch()
    for name in HYDRO_FIELDS + ("phi", "gx", "gy", "gz"):
        set_global_field(tree, name, out[name])
    if cfg.gravity_per_step:
        p = 8
        set_global_field(tree, "mass", st.mass[p:p + st.nz, p:p + st.n, p:p + st.n].cpu().numpy())
    return RunResult(config=cfg, backend=bk.name, threads=threads, tasks_per_multipole=tasks_per_multipole,
                     tree=tree, records=records, computation_s=total_ns / 1e9,
                     launch_stats=LaunchStats(gpu_launches=_lib.launch_count() - launches0))


def bench_records(result: RunResult) -> list:
    """One row per kernel (fixed order) plus the total row (reference driver.py:192-230)."""
    by_name = {r.name: r for r in result.records}
    rows = []
    for kernel in KERNEL_ORDER + ("total",):
        rec = by_name.get(kernel)
        if rec is None:
            continue
        rows.append(BenchRecord(scenario=result.config.name, backend="cuda", simd_width=WARP_WIDTH,
                                threads=result.threads, tasks_per_multipole=result.tasks_per_multipole,
                                kernel=kernel, count=rec.count, mean_ns=rec.mean_ns, total_ns=rec.total_ns,
                                computation_s=result.computation_s))
    return rows


def write_csv(path: str, rows: list) -> None:
    """Append rows (header when the file is new/empty); UTF-8, LF."""
    need_header = not os.path.exists(path) or os.path.getsize(path) == 0
    with io.open(path, "a", encoding="utf-8", newline="") as fh:
        if need_header:
            fh.write(CSV_HEADER + "\n")
        for row in rows:
            fh.write(row.csv_row() + "\n")


def expected_row_count(scenario_name: str, n_runs: int) -> int:
    kernels = 5 if scenario_name == "rotating-star-proxy" else 3
    return n_runs * (kernels + 1)


def sweep(cfg: ScenarioConfig, thread_list: list, backend_list: list, csv_path: str,
          tasks_per_multipole: int = 1, hydro_kernel: str = "cuda", gravity_kernel: str = "cuda") -> list:
    """One run per (threads, backend) pair, rows appended to csv_path."""
    if not thread_list or not backend_list:
        raise ValueError("thread and backend lists must be non-empty")
    for name in backend_list:
        simd.get_backend(name)
    rows = []
    for threads in thread_list:
        for backend in backend_list:
            rows.extend(bench_records(run_scenario(cfg, backend=backend, threads=threads,
                                                   tasks_per_multipole=tasks_per_multipole,
                                                   hydro_kernel=hydro_kernel, gravity_kernel=gravity_kernel)))
    write_csv(csv_path, rows)
    return rows

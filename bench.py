"""Benchmark: the reference's full timestep (config 5) on B200.

Workload (BASELINE.json config 5, restated in SURVEY.md §8(d)): 128^3-cell
periodic unigrid = 4096 subgrids of 8^3, rotating polytrope (floor 0.05),
gamma 1.4, theta 0.34, eps 0.5, expansion order 1.  One bench step = one
reference timestep (driver.py:163-174): mass = rho*dx^3, 6 x (ghost fill +
cluster aggregation + P2P + M2L), max wave speed + dt, 3 x (ghost fill +
reconstruct + flux + update).  z-slabs over N GPUs (NCCL halo + MAX
all-reduce), strong scaling.

value = subgrids advanced one full timestep per second, whole job
        (4096 * steps / max-over-ranks device time), inputs resident in HBM.
e2e   = same unit through the public host API: every step uploads the state
        from pinned host memory, runs the step and reads the new state and
        gravity back (H2D/D2H inside the timed region).
per_kernel: subgrids/s and mean launch time of every kernel inside the timed
        steps (CUDA events on the launching stream); P2P, which runs beside
        M2L on a side stream there, from a short serial pass.
roofline: M2L (the dominant kernel), algorithmic FLOPs (SURVEY.md §8(d):
        26,800,128 per subgrid at order 1) / mean launch time, against the
        FP64 peak measured in this run by a DFMA microbenchmark (no FP64
        entry exists in MEASURED_PEAKS.json).
cpu_baseline: the C restatement of the reference kernels (oracle/, built
        -march=native on this host) on all host threads, timed on a bounded
        sample of the same workload and extrapolated to a full step.

`--impl reference` times that CPU implementation alone (rank 0) with the same
metric/config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "FP64 subgrids/s per kernel (M2L, P2P, hydro) at 1/2/4/8 B200; % FP64/HBM roofline"
UNIT = "subgrids/s"
M2L_FLOP = {1: 26_800_128, 0: 8_338_944}      # SURVEY.md §8(d), per subgrid
P2P_FLOP = 423_936
# fused reconstruct + flux per subgrid: the 512 interior cells
# reconstruct all 26 directions (1,174 each), the 384 one-layer ring cells only
# the 9 directions their faces read (30 + 9*44 each), plus the flux's 1,275,264
HYDRO_ITER_FLOP = 512 * 1_174 + 384 * (30 + 9 * 44) + 1_275_264   # = 2,039,936
# per-kernel roof and algorithmic work per subgrid: FP64
# kernels against the measured DADD/DMUL issue rate, HBM kernels against the
# measured copy bandwidth (update: U interior read + write + the three flux
# arrays; wave speed: the U interior)
KERNEL_ROOF = {"m2l": ("fp64", M2L_FLOP[1]), "p2p": ("fp64", P2P_FLOP), "hydro_fused": ("fp64", HYDRO_ITER_FLOP),
               "hydro_update": ("hbm", 2 * 5 * 512 * 8 + 5 * (576 * 3) * 8), "max_wavespeed": ("hbm", 5 * 512 * 8)}
LEVEL = 4
PER_KERNEL_STEPS = 2  # steps of the serial pass that times P2P alone


def config_dict(world: int) -> dict:
    return {"workload": "config5: full timestep, 128^3 unigrid (4096 subgrids of 8^3), 6x(P2P+M2L) + 3x hydro",
            "level": LEVEL, "subgrids": 8 ** LEVEL, "theta": 0.34, "eps": 0.5, "expansion_order": 1,
            "gamma": 1.4, "floor": 0.05, "omega": 0.1, "parallelism": f"zslab{world}",
            "l2": "per-step working set > L2 (fluxes 283 MB written+read per hydro iteration, state 92 MB); "
                  "no explicit flush"}


# -- clocks ---------------------------------------------------------------------

REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class ClockSampler:
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.out = None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm,power.draw," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        self.out = out

    def summary(self) -> dict:
        if not self.out:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons, power = [], [], set(), []
        for line in self.out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 3 + len(REASONS):
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for r, v in zip(REASONS, f[3:]):
                if v.lower().startswith("active"):
                    reasons.add(r)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# -- CPU baseline (oracle) --------------------------------------------------------

def cpu_sample(state: dict, level: int, threads: int, m2l_leaves: int) -> dict:
    """Time the CPU restatement of the reference kernels on a bounded sample
    of the config-5 workload; return per-kernel rates and the extrapolated
    full-step rate (subgrids/s)."""
    from oracle import oracle as O
    n = 8 << level
    dx = 1.0 / n
    allc = O.leaf_coords(level)
    rng = np.random.default_rng(5)
    U = np.stack([state[k] for k in O.HYDRO_FIELDS])
    mass = U[0] * dx ** 3
    pick = np.ascontiguousarray(allc[rng.choice(len(allc), size=min(m2l_leaves, len(allc)), replace=False)])
    sample512 = np.ascontiguousarray(allc[rng.choice(len(allc), size=512, replace=False)])
    t = {}
    w0 = time.perf_counter()
    t0 = time.perf_counter()
    O.m2l_batch(mass, dx, 0.34, 0.5, 1, pick, threads)
    t["m2l"] = len(pick) / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    O.p2p_batch(mass, dx, 0.34, 0.5, sample512, threads)
    t["p2p"] = 512 / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    O.wavespeed_batch(U, 1.4, 1e-12, sample512, threads)
    t["max_wavespeed"] = 512 / (time.perf_counter() - t0)
    t0 = time.perf_counter()
    O.hydro_batch(U, 1e-12, 1.4, 1e-4, sample512, threads)
    t["hydro"] = 512 / (time.perf_counter() - t0)
    wall = time.perf_counter() - w0
    nl = len(allc)
    step_s = 6 * (nl / t["m2l"] + nl / t["p2p"]) + nl / t["max_wavespeed"] + 3 * nl / t["hydro"]
    return {"rates": t, "step_s": step_s, "value": nl / step_s, "extrapolated": True,
            "sampled_leaves": {"m2l": len(pick), "p2p": 512, "max_wavespeed": 512, "hydro": 512},
            "sample_wall_s": wall,
            "omitted_phases": ["mass = rho*dx^3", "cluster_aggregate (inside the port's M2L per leaf)",
                               "ghost exchange (9 per step)", "dt reduction"],
            "sample": f"M2L on {len(pick)} random leaves, P2P/wavespeed/hydro iteration on 512 leaves of "
                      f"the config-5 state; full 4096-leaf step extrapolated as 6*(M2L+P2P)+ws+3*hydro "
                      f"(hydro sample at a fixed dt/dx of 1e-4)"}


def numba_reference_sample(state: dict, level: int, threads: int, m2l_leaves: int) -> dict:
    """The reference itself (simdgrid, numba compiled path, installed in
    baseline/_ref by `pip install --target`) on a bounded sample of the same
    config-5 workload, through its own WorkerPool (runtime.py:180-278, one
    task per leaf as driver.py:164-174 spawns them) and public kernel entry
    points (kernels/__init__.py:122-267): per-leaf M2L/P2P/hydro on sampled
    leaves, the ghost exchanges and the wave-speed pass in full, extrapolated
    to one 4096-leaf step.  Numba JIT compilation happens in an untimed
    warm-up call of every kernel."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "simdgrid").is_dir():
        return {"available": False, "why": "baseline/_ref/simdgrid not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sg_numba_cache")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from simdgrid import kernels as RK
        from simdgrid.octree import build_unigrid, exchange_ghosts, neighborhood27
        from simdgrid.runtime import WorkerPool
    except Exception as exc:  # numba missing etc.
        return {"available": False, "why": f"import failed: {exc}"}
    w0 = time.perf_counter()
    tree = build_unigrid(level)
    for leaf in tree.leaves:
        cx, cy, cz = leaf.coord
        sl = (slice(cz * 8, cz * 8 + 8), slice(cy * 8, cy * 8 + 8), slice(cx * 8, cx * 8 + 8))
        for name in ("rho", "sx", "sy", "sz", "E"):
            leaf.interior(name)[...] = state[name][sl]
    h = RK.HydroConfig(gamma=1.4)
    g = RK.GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    nl = len(tree.leaves)
    rng = np.random.default_rng(5)
    pick = [int(i) for i in rng.choice(nl, size=min(m2l_leaves, nl), replace=False)]
    s512 = [int(i) for i in rng.choice(nl, size=min(512, nl), replace=False)]
    t = {}

    def gravity_job(i, which):
        src = neighborhood27(tree, i)
        if which == "p2p":
            RK.monopole_kernel(tree.leaves[i], src, g, "scalar")
        else:
            RK.multipole_kernel(tree.leaves[i], src, g, "scalar")

    with WorkerPool(threads) as pool:
        def run(fn, ids, *a):
            futs = [pool.spawn(fn, i, *a) for i in ids]
            for f in futs:
                f.result()
        tc = time.perf_counter()
        for leaf in tree.leaves:
            leaf.interior("mass")[...] = leaf.interior("rho") * leaf.dx ** 3
        t["set_mass_s"] = time.perf_counter() - tc
        tc = time.perf_counter()
        exchange_ghosts(tree, "gravity")
        t["exchange_gravity_s"] = time.perf_counter() - tc
        tc = time.perf_counter()
        exchange_ghosts(tree, "hydro")
        t["exchange_hydro_s"] = time.perf_counter() - tc
        # untimed JIT warm-up of every kernel on one leaf
        gravity_job(0, "p2p")
        gravity_job(0, "m2l")
        s0 = RK.max_wavespeed(tree.leaves[0], h)
        RK.flux(tree.leaves[0], RK.reconstruct(tree.leaves[0], h, "scalar"), h, "scalar")
        tc = time.perf_counter()
        s_pre = max(RK.max_wavespeed(leaf, h) for leaf in tree.leaves)   # driver.py:170 (serial)
        t["max_wavespeed_s"] = time.perf_counter() - tc
        dt = h.cfl * tree.dx / (3.0 * s_pre)
        tc = time.perf_counter()
        run(gravity_job, s512, "p2p")
        t["p2p_per_leaf_s"] = (time.perf_counter() - tc) / len(s512)
        tc = time.perf_counter()
        run(gravity_job, pick, "m2l")
        t["m2l_per_leaf_s"] = (time.perf_counter() - tc) / len(pick)

        def hydro_job(i):
            leaf = tree.leaves[i]
            q = RK.reconstruct(leaf, h, "scalar")
            fl = RK.flux(leaf, q, h, "scalar")
            RK.hydro_update(leaf, fl, dt, h)
        tc = time.perf_counter()
        run(hydro_job, s512)
        t["hydro_per_leaf_s"] = (time.perf_counter() - tc) / len(s512)
    del s0
    step_s = (t["set_mass_s"] + 6 * (t["exchange_gravity_s"] + nl * (t["p2p_per_leaf_s"] + t["m2l_per_leaf_s"]))
              + t["max_wavespeed_s"] + 3 * (t["exchange_hydro_s"] + nl * t["hydro_per_leaf_s"]))
    return {"available": True, "value": nl / step_s, "unit": UNIT, "cores": threads, "kind": "reference",
            "step_s": step_s, "extrapolated": True, "parts": t, "sample_wall_s": time.perf_counter() - w0,
            "sampled_leaves": {"m2l": len(pick), "p2p": len(s512), "hydro": len(s512), "max_wavespeed": nl},
            "sample": f"reference simdgrid (numba) via WorkerPool({threads}): M2L on {len(pick)} random leaves, "
                      f"P2P and hydro iteration (reconstruct+flux+update at the step's dt) on {len(s512)}; "
                      f"set_mass, ghost exchanges and the serial wave-speed pass over all {nl} leaves; "
                      f"step extrapolated as set_mass + 6*(exchange + nl*(P2P+M2L)) + ws + "
                      f"3*(exchange + nl*hydro)"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2210_06439_b200 import scenarios
    kind = "port-native" if O.use_native() else "port"
    threads = O.max_threads()
    state = scenarios.config5_state(LEVEL)
    m2l_leaves = max(48 * threads, 64)
    for _ in range(args.warmup):
        cpu_sample(state, LEVEL, threads, m2l_leaves)
    vals, steps = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_sample(state, LEVEL, threads, m2l_leaves)
        vals.append(r["value"])
        steps.append(r["step_s"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    numba = numba_reference_sample(state, LEVEL, threads, max(8 * threads, 32))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.median(steps) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (config-5 IC)",
        "impl": "reference",
        "config": config_dict(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "build": kind, "sample": r["sample"], "rates": r["rates"],
                         "extrapolated": True, "sampled_leaves": r["sampled_leaves"],
                         "sample_wall_s": r["sample_wall_s"],
                         "omitted_phases": r["omitted_phases"], "wall_s_timed": wall},
        "extrapolated": True,
        "reference_numba": numba,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference arm = the oracle's C restatement of the reference numba kernels "
                "(bit-identical to it, tests/test_oracle_golden.py), all host threads; each step's time "
                "is EXTRAPOLATED from a bounded sample (wall_s_timed is the real time of the timed samples); "
                "reference_numba = the reference package itself on the same kind of sample",
    }
    print(json.dumps(_strict_json(line), allow_nan=False), flush=True)


def _strict_json(obj):
    """Non-finite floats -> null, so every printed line is strict JSON."""
    if isinstance(obj, float):
        return obj if math.isfinite(obj) else None
    if isinstance(obj, dict):
        return {k: _strict_json(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_strict_json(v) for v in obj]
    return obj


# -- our arm ------------------------------------------------------------------------

def m2l_traffic_from_profile():
    """dram__bytes_read.sum + dram__bytes_write.sum of one M2L launch at
    level 4, from the committed ncu --set full summary (profiles/)."""
    import re
    for f in sorted((REPO / "profiles").glob("r*_m2l_L4_ncu_full.txt"), reverse=True):
        # one section per captured kernel; take the exact M2L one
        for txt in f.read_text().split("== ncu --set full")[1:]:
            name = re.search(r"Kernel Name\s+(.*)", txt)
            if not name or not ("m2l_kernel" in name.group(1) or "m2l_pair_kernel" in name.group(1)):
                continue
            vals = {}
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                m = re.search(key + r"\s+([0-9.]+)\s+(\w+)", txt)
                if m:
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(2), 1)
                    vals[key] = float(m.group(1)) * scale
            if len(vals) == 2:
                return sum(vals.values()), f.name
    return None, None


def fp64_peak(torch) -> dict:
    import ctypes

    from paper_2210_06439_b200 import _lib
    L = _lib.load()
    sink = torch.zeros(1, dtype=torch.float64, device="cuda")
    res = {}
    for mode, name in ((0, "dfma_tflops"), (1, "dadd_tflops")):
        best = 0.0
        for rep in range(4):
            flops = ctypes.c_int64()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            rc = L.sg_fp64_peak(mode, 2000, sink.data_ptr(), ctypes.byref(flops),
                                torch.cuda.current_stream().cuda_stream)
            e.record()
            torch.cuda.synchronize()
            if rc:
                raise RuntimeError(L.sg_last_error().decode())
            if rep:
                best = max(best, flops.value / (s.elapsed_time(e) * 1e-3) / 1e12)
        res[name] = best
    return res


def per_config_rates(torch, peaks: dict) -> dict:
    """Per-kernel device rates on BASELINE configs 1-4 (SURVEY.md 8(d)
    restatements), median of 5 CUDA-event timed launches after a warm-up;
    inputs resident, host enqueue hidden.  FP64 fractions are against the measured DADD issue peak
    (the attainable roof without FMA contraction); reconstruct's against HBM."""
    import statistics as stats

    from paper_2210_06439_b200 import batched as B
    from paper_2210_06439_b200 import grid, scenarios
    from paper_2210_06439_b200.batched import View
    from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig

    def timed(fn, reps=5, trimmed=False):
        """device time of fn (median of reps); trimmed=True: 10%-trimmed mean,
        for microsecond-scale calls (event timestamps tick every 1.024 us on
        these boxes, so a median of a few reps is quantised)"""
        fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)  # GPU busy while the host enqueues: device time only
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        if trimmed:
            return stats.mean(sorted(ts)[reps // 10:reps - reps // 10])
        return stats.median(ts)

    issue = peaks["dadd_tflops"] * 1e12
    hbm = None
    try:
        hbm = json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
    except Exception:
        pass
    out = {}
    g1 = GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    # config 1: one 24^3 neighbourhood (cluster aggregation + the fused
    # latency-mode M2L: 64 two-CTA clusters)
    cube = torch.from_numpy(scenarios.config1_cube(0)).cuda()
    cl = torch.empty((12, 12, 12, 4), dtype=torch.float64, device="cuda")
    res = torch.empty((4, 8, 8, 8), dtype=torch.float64, device="cuda")
    dx = 1.0 / 64
    rad = dx / 0.34
    eps = 0.5 * dx

    def c1():
        B.cluster_aggregate(cube, dx, cl)
        B.m2l(cube, View(8, 8, 8, 8), cl, 0, None, 1, dx, rad * rad, eps * eps, 1, res, View(8, 8, 8, 0))
    t = timed(c1, reps=40, trimmed=True)
    out["config1_m2l_single"] = {"latency_us": t * 1e6, "subgrids_per_s": 1 / t,
                                 "timing": "10%-trimmed mean of 40 reps (CUDA event ticks are 1.024 us)"}
    # configs 2-4 on the 512-subgrid level-3 grid
    u = grid.UnigridState(3, HydroConfig(gamma=5.0 / 3.0), g1)
    z = np.zeros((64, 64, 64))
    for name, rho in (("config2_p2p", scenarios.config2_rho(1, 3)), ("config3_m2l", scenarios.config3_rho(3))):
        u.load({"rho": rho, "sx": z, "sy": z, "sz": z, "E": rho})
        u.set_mass()
        u._halo(u.mass, 1, u.mv)
        B.cluster_aggregate(u.mass, u.dx, u.clusters)
        if name == "config2_p2p":
            t = timed(lambda: B.p2p(u.mass, u.mv, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, u.halo, u.grav, u.gv))
            flop = P2P_FLOP
        else:
            t = timed(lambda: B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, 1,
                                    u.grav, u.gv))
            flop = M2L_FLOP[1]
        out[name] = {"ms": t * 1e3, "subgrids_per_s": 512 / t, "tflops": flop * 512 / t / 1e12,
                     "frac_fp64_issue": flop * 512 / t / issue}
    u.load(scenarios.config4_state(3))
    u._halo(u.U, 5, u.uv)
    tf = timed(lambda: B.hydro_fused(u.U, u.uv, u.leaves, u.nleaves, 1e-12, 5.0 / 3.0, u.FX, u.FY, u.FZ, u.smax,
                                     u.flux_err))
    tr = timed(lambda: B.reconstruct(u.U, u.uv, u.leaves, u.nleaves, 1e-12, u.Q))
    tx = timed(lambda: B.flux(u.Q, u.nleaves, 5.0 / 3.0, u.FX, u.FY, u.FZ, u.smax, u.flux_err))
    rec = {"fused_ms": tf * 1e3, "subgrids_per_s": 512 / tf,
           "fused_frac_fp64_issue": HYDRO_ITER_FLOP * 512 / tf / issue,
           "reconstruct_ms": tr * 1e3, "flux_ms": tx * 1e3, "unfused_subgrids_per_s": 512 / (tr + tx)}
    if hbm:
        rec["reconstruct_frac_hbm"] = 1_109_120 * 512 / tr / hbm
        rec["flux_frac_hbm"] = 1_109_128 * 512 / tx / hbm
    out["config4_hydro"] = rec
    return out


def alt_precision_run(torch, dist, args, state, slab, group, peaks, world, barrier) -> dict:
    """The other gravity precision on the same workload: timed steps, M2L
    roofline, and its deviation from the exact path on one gravity pass
    (max-norm relative per component, and elementwise statistics)."""
    from paper_2210_06439_b200 import grid
    from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig
    prec = "fma" if args.precision == "exact" else "exact"
    g = GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    u = grid.UnigridState(LEVEL, HydroConfig(gamma=1.4), g, slab=slab, group=group, precision=prec)
    u.load(state)
    for _ in range(args.warmup):
        u.step()
    u.load(state)
    barrier()
    u.timers = {}
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record()
    for _ in range(args.steps):
        u.step()
    e_ev.record()
    barrier()
    el = torch.tensor([s_ev.elapsed_time(e_ev) * 1e-3], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    u.check_errors()
    m2l = [a.elapsed_time(b) * 1e-3 for a, b in u.timers["m2l"]]
    m2l_s = sum(m2l) / len(m2l)
    u.timers = None
    # accuracy of fma vs exact on one gravity pass of the initial state
    outs = {}
    for p in ("exact", "fma"):
        v = grid.UnigridState(LEVEL, HydroConfig(gamma=1.4), g, slab=slab, group=group, precision=p)
        v.load(state)
        v.set_mass()
        v.gravity_iteration()
        outs[p] = v.grav.cpu().numpy()
    acc = {}
    for c, name in enumerate(("phi", "gx", "gy", "gz")):
        a, b = outs["fma"][c], outs["exact"][c]
        d = np.abs(a - b)
        rel = d / np.maximum(np.abs(b), 1e-300)
        acc[name] = {"maxnorm_rel": float(d.max() / np.abs(b).max()), "elem_rel_max": float(rel.max()),
                     "frac_elem_rel_gt_1e-12": float((rel > 1e-12).mean())}
    achieved = M2L_FLOP[1] * u.nleaves / m2l_s / 1e12
    return {"precision": prec, "value": 8 ** LEVEL * args.steps / el.item(),
            "ms_per_step": el.item() * 1e3 / args.steps, "m2l_mean_ms": m2l_s * 1e3,
            "roofline": {"kernel": "m2l", "achieved": achieved, "unit": "TFLOP/s", "peak": peaks["dfma_tflops"],
                         "frac": achieved / peaks["dfma_tflops"], "frac_issue": achieved / peaks["dadd_tflops"]},
            "deviation_fma_vs_exact": acc,
            "note": "hydro is bit-exact in both modes; only gravity (M2L, P2P) arithmetic differs"}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2210_06439_b200 import _lib, grid, scenarios
    from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig
    from paper_2210_06439_b200.slab import Slab

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and local >= torch.cuda.device_count():
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPU(s) visible")
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        # NCCL's own init lines (communicator, rank -> GPU, transport) on
        # stderr, so a run's rank count is visible independently of our JSON
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if dist.get_world_size() != world:
            raise SystemExit(f"process group has {dist.get_world_size()} ranks, WORLD_SIZE={world}")
    slab = Slab(LEVEL, rank, world)
    state = scenarios.config5_state(LEVEL)
    peaks = fp64_peak(torch)
    try:
        hbm_peak = json.loads((REPO / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
    except Exception:
        hbm_peak = 6553.0e9  # B200_PROFILING.md fallback (of fallback)

    u = grid.UnigridState(LEVEL, HydroConfig(gamma=1.4), GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                          slab=slab, group=group, precision=args.precision)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    u.load(state)
    for _ in range(args.warmup):
        u.step()
    u.check_errors()
    u.load(state)
    barrier()
    gpu_uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    uuids = [gpu_uuid]
    if world > 1:  # one distinct GPU per rank, or the scaling numbers mean nothing
        uuids = [None] * world
        dist.all_gather_object(uuids, gpu_uuid)
    gpus_active = len(set(uuids))
    u.timers = {}
    launches0 = _lib.launch_count()
    with ClockSampler(gpu_uuid) as clk:
        s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_ev.record()
        for _ in range(args.steps):
            u.step()
        e_ev.record()
        barrier()
    launches = _lib.launch_count() - launches0
    elapsed = s_ev.elapsed_time(e_ev) * 1e-3
    u.check_errors()
    # P2P runs beside M2L on a side stream in the timed steps (grid.py
    # gravity_kernels), where an event pair would time its wait for the M2L
    # tail: its standalone launch time comes from a short serial pass
    timers, overlap = u.timers, u.overlap_p2p
    u.load(state)
    barrier()
    u.timers, u.overlap_p2p = {}, False
    for _ in range(min(args.steps, PER_KERNEL_STEPS)):
        u.step()
    barrier()
    u.check_errors()
    timers["p2p"] = u.timers["p2p"]
    u.timers, u.overlap_p2p = timers, overlap
    per_kernel = {}
    for name, evs in u.timers.items():
        ts = [a.elapsed_time(b) * 1e-3 for a, b in evs]
        per_kernel[name] = {"launches": len(ts), "mean_ms": 1e3 * sum(ts) / len(ts),
                            "subgrids_per_s": u.nleaves * world * len(ts) / sum(ts)}
        if name in KERNEL_ROOF:  # per GPU: this rank's subgrids over its own launch time
            bound, work = KERNEL_ROOF[name]
            rate = u.nleaves * len(ts) / sum(ts)
            if bound == "fp64":
                per_kernel[name]["roofline"] = {"bound": "fp64", "tflops": work * rate / 1e12,
                                                "frac_fp64_issue": work * rate / (peaks["dadd_tflops"] * 1e12),
                                                "frac_dfma_peak": work * rate / (peaks["dfma_tflops"] * 1e12)}
            elif hbm_peak:
                per_kernel[name]["roofline"] = {"bound": "hbm", "gbs": work * rate / 1e9,
                                                "frac_hbm": work * rate / hbm_peak}
    u.timers = None
    t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed = t.item()
    total_leaves = 8 ** LEVEL
    value = total_leaves * args.steps / elapsed

    # e2e through the public host API (grid.HostPipeline): every step uploads
    # its input state from pinned host memory and reads the new state and
    # gravity back into pinned host memory; transfers overlap compute on a
    # copy stream (double-buffered staging); timed until the last readback
    host_in = torch.from_numpy(np.ascontiguousarray(
        np.stack([state[k][slab.z0:slab.z0 + slab.nz] for k in ("rho", "sx", "sy", "sz", "E")]))).pin_memory()
    host_out = [torch.empty((9, slab.nz, slab.n, slab.n), dtype=torch.float64).pin_memory() for _ in range(2)]
    pipe = grid.HostPipeline(u)
    e2e_steps = max(1, args.steps)
    for j in range(2):  # warm the pipeline (streams, events, staging)
        pipe.submit(host_in, host_out[j % 2])
    pipe.synchronize()
    barrier()
    t0 = time.perf_counter()
    for j in range(e2e_steps):
        pipe.submit(host_in, host_out[j % 2])
    pipe.synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    u.check_errors()
    ref_out = grid.UnigridState(LEVEL, HydroConfig(gamma=1.4), GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                                slab=slab, group=group, precision=args.precision) if args.verify_e2e else None
    if ref_out is not None:  # the pipelined result equals load + step + fetch
        ref_out.load(state)
        ref_out.step()
        f = ref_out.fetch()
        want = np.stack([f[k] for k in ("rho", "sx", "sy", "sz", "E", "phi", "gx", "gy", "gz")])
        assert np.array_equal(host_out[(e2e_steps - 1) % 2].numpy(), want), "pipelined e2e result differs"
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = t.item()
    cells = slab.nz * slab.n * slab.n
    h2d = 5 * cells * 8 * world
    d2h = 9 * cells * 8 * world

    m2l = per_kernel.get("m2l", {})
    m2l_ms = m2l.get("mean_ms", float("nan"))
    achieved = M2L_FLOP[1] * u.nleaves / (m2l_ms * 1e-3) / 1e12
    roofline = {"kernel": "m2l", "bound": "fp64", "achieved": achieved, "unit": "TFLOP/s",
                "peak": peaks["dfma_tflops"], "frac": achieved / peaks["dfma_tflops"],
                "peak_source": "measured in this run: DFMA microbenchmark (sg_fp64_peak); FMA counted as 2 FLOP",
                "peak_issue": peaks["dadd_tflops"], "frac_issue": achieved / peaks["dadd_tflops"],
                "flop_per_subgrid": M2L_FLOP[1], "subgrids_per_launch": u.nleaves}
    traffic, src = m2l_traffic_from_profile()
    roofline["traffic"] = traffic if u.nleaves == 4096 else None
    roofline["traffic_unit"] = "bytes/launch (DRAM read+write, ncu)"
    roofline["traffic_source"] = f"profiles/{src}" if src else None
    roofline["note"] = ("FP64 CUDA-core bound (not hbm/tensor): parity forbids FMA contraction, so the "
                        "attainable ceiling is the DADD/DMUL issue rate (frac_issue); traffic << algorithmic "
                        "bytes because the neighbourhoods are re-read from L2")

    alt = None
    if not args.no_alt:
        alt = alt_precision_run(torch, dist, args, state, slab, group, peaks, world, barrier)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "gpus_active": gpus_active,
        "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "precision": args.precision,
        "comm": ({"backend": "nccl", "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                  "ranks": world, "per_step": "6 mass + 3 U z-halo exchanges (2 sends + 2 recvs each), "
                  "1 MAX all-reduce"} if world > 1 else None),
        "data": "synthetic config-5 IC (seedless, deterministic)",
        "config": config_dict(world),
        "e2e": {"value": total_leaves * e2e_steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "per_kernel": per_kernel,
        "roofline": roofline,
    }
    if alt is not None:
        line["alt_precision"] = alt
    if rank == 0:
        line["clocks"] = clk.summary()
        try:
            line["per_config"] = per_config_rates(torch, peaks)
        except Exception as exc:  # informational; never fails the headline
            line["per_config"] = {"error": str(exc)}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as O
            kind = "port-native" if O.use_native() else "port"
            threads = O.max_threads()
            r = cpu_sample(state, LEVEL, threads, max(48 * threads, 64))
            line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": threads, "kind": "port",
                                    "build": kind, "sample": r["sample"], "rates": r["rates"],
                                    "extrapolated": True, "sampled_leaves": r["sampled_leaves"],
                                    "sample_wall_s": r["sample_wall_s"], "omitted_phases": r["omitted_phases"]}
            if not args.no_numba:
                line["cpu_baseline"]["reference_numba"] = numba_reference_sample(
                    state, LEVEL, threads, max(8 * threads, 32))
        except Exception as exc:  # the baseline is a report, never the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                    "sample": f"failed: {exc}"}
    if rank == 0:
        print(json.dumps(_strict_json(line), allow_nan=False), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--verify-e2e", action="store_true", help="check the pipelined e2e result bitwise")
    ap.add_argument("--precision", choices=["exact", "fma"], default="exact",
                    help="gravity arithmetic of the headline run: exact = bit-identical to the reference "
                         "(default); fma = FMA-contracted, within 1e-12 max-norm per component")
    ap.add_argument("--no-alt", action="store_true", help="skip the secondary-precision measurement")
    ap.add_argument("--no-numba", action="store_true", help="skip the reference-package (numba) CPU sample")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    env_world = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        run_reference(args)
        return
    if env_world is None and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    world = int(env_world or "1")
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a different "
              f"GPU count", file=sys.stderr)
        sys.exit(2)
    run_ours(args)


def relaunch(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1 and return its exit code.
    Fails loudly when the node has fewer than N GPUs."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} requested but only {have} CUDA device(s) visible", file=sys.stderr)
        return 3
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    print("bench.py: launching " + " ".join(cmd[2:]), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


if __name__ == "__main__":
    main()

"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
(``simdgrid`` from /root/reference/pkg/src, numba-compiled production path).

Run once in the build container (the reference is not present on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [--skip-l4]

Fixtures record inputs (when small) or input digests (when generated from a
seed by paper_2210_06439_b200.scenarios), the reference's outputs as full
arrays or SHA-256 digests of their float64 bytes, and floats as hex strings.
The oracle (oracle/) and the CUDA path are both checked against these.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from simdgrid import kernels as K  # noqa: E402  (the reference)
from simdgrid.kernels import compiled  # noqa: E402
from simdgrid.octree import build_unigrid, exchange_ghosts, neighborhood27  # noqa: E402

from paper_2210_06439_b200 import scenarios  # noqa: E402

FIELDS = ("rho", "sx", "sy", "sz", "E")
POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 4)


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def fhex(x: float) -> str:
    return float(x).hex()


def tree_from_global(level: int, fields: dict[str, np.ndarray]):
    tree = build_unigrid(level)
    for leaf in tree.leaves:
        cx, cy, cz = leaf.coord
        sl = (slice(cz * 8, cz * 8 + 8), slice(cy * 8, cy * 8 + 8), slice(cx * 8, cx * 8 + 8))
        for name, arr in fields.items():
            leaf.interior(name)[...] = arr[sl]
    return tree


def global_from_tree(tree, name: str) -> np.ndarray:
    n = tree.leaves_per_axis * 8
    out = np.empty((n, n, n))
    for leaf in tree.leaves:
        cx, cy, cz = leaf.coord
        out[cz * 8:(cz + 1) * 8, cy * 8:(cy + 1) * 8, cx * 8:(cx + 1) * 8] = leaf.interior(name)
    return out


def leaf_key(leaf) -> str:
    return "%d,%d,%d" % leaf.coord


# ---------------------------------------------------------------------------

def gravity_cfg1():
    """Config 1: single 24^3 neighbourhood, compiled kernels called exactly as
    multipole_prepare does (kernels/__init__.py:224-244)."""
    cube = scenarios.config1_cube(0)
    dx = 1.0 / 64
    out = {"cube": cube}
    for theta in (0.34, 0.5):
        rad = dx / theta
        rad2 = rad * rad
        epsd = 0.5 * dx
        eps2 = epsd * epsd
        M, Dx, Dy, Dz = compiled.cluster_aggregate(cube, dx)
        if theta == 0.34:
            out["M"], out["Dx"], out["Dy"], out["Dz"] = M, Dx, Dy, Dz
        for order in (0, 1):
            res = np.zeros((4, 8, 8, 8))
            compiled.multipole_kernel_impl(cube, M, Dx, Dy, Dz, dx, rad2, eps2, order, 1, 0, 512,
                                           res[0], res[1], res[2], res[3])
            out[f"m2l_t{int(theta * 100)}_o{order}"] = res
        # P2P over the central (8+2h)^3 of the same cube
        halo = K.gravity_halo(theta)
        sub = np.ascontiguousarray(cube[8 - halo:16 + halo, 8 - halo:16 + halo, 8 - halo:16 + halo])
        res = np.zeros((4, 8, 8, 8))
        compiled.monopole_kernel_impl(sub, dx, rad2, eps2, halo, 1, res[0], res[1], res[2], res[3])
        out[f"p2p_t{int(theta * 100)}"] = res
    np.savez_compressed(HERE / "gravity_cfg1.npz", **out)


def random_mass_global(rng, level: int) -> np.ndarray:
    """tests/util.py:43-50 restated on a global field (uniform masses,
    5% zeros, times dx^3), filled leaf by leaf in Morton order."""
    tree = build_unigrid(level)
    n = 8 << level
    g = np.empty((n, n, n))
    for leaf in tree.leaves:
        m = rng.uniform(0.0, 1.0, (8, 8, 8))
        m[rng.uniform(size=(8, 8, 8)) < 0.05] = 0.0
        cx, cy, cz = leaf.coord
        g[cz * 8:(cz + 1) * 8, cy * 8:(cy + 1) * 8, cx * 8:(cx + 1) * 8] = m * leaf.dx**3
    return g


def gravity_tree():
    """L=1 random mass tree through the reference API (monopole_kernel /
    multipole_kernel), every leaf, several theta / orders."""
    rng = np.random.default_rng(77)
    mass = random_mass_global(rng, 1)
    tree = tree_from_global(1, {"mass": mass})
    out = {"mass": mass}
    cases = [("p2p", 0.5, 0), ("p2p", 0.34, 0), ("p2p", 0.2, 0),
             ("m2l", 0.34, 0), ("m2l", 0.34, 1), ("m2l", 0.5, 1), ("m2l", 0.2, 1)]
    for kind, theta, order in cases:
        cfg = K.GravityConfig(theta=theta, eps=0.5, expansion_order=order)
        res = np.zeros((len(tree.leaves), 4, 8, 8, 8))
        coords = np.zeros((len(tree.leaves), 3), dtype=np.int64)

        def job(i):
            t = tree.leaves[i]
            src = neighborhood27(tree, i)
            # private copies of the output fields: jobs run concurrently
            fn = K.monopole_kernel if kind == "p2p" else K.multipole_kernel
            outs = fn(t, src, cfg, "scalar")
            return i, [np.array(a) for a in outs]

        for i, outs in POOL.map(job, range(len(tree.leaves))):
            res[i] = np.stack(outs)
            coords[i] = tree.leaves[i].coord
        out[f"{kind}_t{int(theta * 100)}_o{order}"] = res
    out["coords"] = coords
    np.savez_compressed(HERE / "gravity_tree.npz", **out)


def batched_gravity(level, mass, kind, theta, order):
    """Run the reference API over every leaf; return global (4,n,n,n) output."""
    tree = tree_from_global(level, {"mass": mass})
    cfg = K.GravityConfig(theta=theta, eps=0.5, expansion_order=order)

    def job(i):
        t = tree.leaves[i]
        fn = K.monopole_kernel if kind == "p2p" else K.multipole_kernel
        fn(t, neighborhood27(tree, i), cfg, "scalar")

    list(POOL.map(job, range(len(tree.leaves))))
    return np.stack([global_from_tree(tree, nm) for nm in ("phi", "gx", "gy", "gz")])


def per_leaf_digests(level, out4):
    """digest of out4[:, leaf block] for every leaf, keyed 'cx,cy,cz'."""
    na = 1 << level
    d = {}
    for cz in range(na):
        for cy in range(na):
            for cx in range(na):
                blk = out4[:, cz * 8:(cz + 1) * 8, cy * 8:(cy + 1) * 8, cx * 8:(cx + 1) * 8]
                d["%d,%d,%d" % (cx, cy, cz)] = digest(blk)
    return d


def cfg2_p2p(man):
    level = 3
    dx = 1.0 / 64
    rho = scenarios.config2_rho(1, level)
    mass = rho * dx**3
    out = batched_gravity(level, mass, "p2p", 0.34, 0)
    man["cfg2_p2p"] = {
        "level": level, "seed": 1, "theta": 0.34, "eps": 0.5,
        "input_digest": digest(rho),
        "output_digest": digest(out),
        "field_digests": [digest(out[i]) for i in range(4)],
        "leaf_digests": per_leaf_digests(level, out),
    }
    np.savez_compressed(HERE / "cfg2_p2p_leaf0.npz", out=out[:, :8, :8, :8])


def cfg3_m2l(man):
    level = 3
    dx = 1.0 / 64
    rho = scenarios.config3_rho(level)
    mass = rho * dx**3
    rec = {"level": level, "theta": 0.34, "eps": 0.5, "input_digest": digest(rho)}
    for order in (1, 0):
        t0 = time.time()
        out = batched_gravity(level, mass, "m2l", 0.34, order)
        print(f"  cfg3 order {order}: {time.time() - t0:.1f}s", flush=True)
        rec[f"o{order}"] = {
            "output_digest": digest(out),
            "field_digests": [digest(out[i]) for i in range(4)],
            "leaf_digests": per_leaf_digests(level, out),
        }
        if order == 1:
            np.savez_compressed(HERE / "cfg3_m2l_leaf_center.npz", out=out[:, 24:32, 24:32, 24:32])
    man["cfg3_m2l"] = rec


def cfg4_hydro(man):
    level = 3
    st = scenarios.config4_state(level)
    tree = tree_from_global(level, st)
    exchange_ghosts(tree, "hydro")
    h = K.HydroConfig(gamma=5.0 / 3.0)

    def job(i):
        leaf = tree.leaves[i]
        q = K.reconstruct(leaf, h, "scalar")
        fl = K.flux(leaf, q, h, "scalar")
        return leaf_key(leaf), digest(q.values), (digest(fl.fx), digest(fl.fy), digest(fl.fz)), fl.max_speed

    recs = {}
    smax = 0.0
    for key, qd, fd, s in POOL.map(job, range(len(tree.leaves))):
        recs[key] = {"q": qd, "fx": fd[0], "fy": fd[1], "fz": fd[2], "smax": fhex(s)}
        smax = max(smax, s)
    man["cfg4_hydro"] = {
        "level": level, "gamma": fhex(5.0 / 3.0),
        "input_digest": digest(np.stack([st[k] for k in FIELDS])),
        "smax": fhex(smax), "leaves": recs,
    }


def random_hydro_block(rng, gamma=1.4):
    """tests/util.py:16-30 restated as a (5,12,12,12) array."""
    scale = float(2.0 ** rng.integers(-6, 7))
    shape = (12, 12, 12)
    rho = (1.0 + 0.1 * rng.uniform(-1.0, 1.0, shape)) * scale
    v = 0.1 * rng.uniform(-1.0, 1.0, (3, *shape))
    p = (1.0 + 0.1 * rng.uniform(-1.0, 1.0, shape)) * scale
    E = p / (gamma - 1.0) + 0.5 * rho * (v**2).sum(axis=0)
    return np.stack([rho, rho * v[0], rho * v[1], rho * v[2], E])


def hydro_random():
    """Per-subgrid hydro kernels on random blocks + error and floor cases."""
    from simdgrid.kernels.geometry import DIR_MINUS, DIR_PLUS, DIRECTIONS_F, SIMPSON_W

    rng = np.random.default_rng(2024)
    out = {}
    blocks = [random_hydro_block(rng) for _ in range(4)]
    # a block whose energy is clamped (tests/test_hydro_kernels.py:88-97)
    b = random_hydro_block(rng)
    b[4] *= 0.01
    blocks.append(b)
    # a geometric density ramp that engages the rho floor (67-77)
    base = np.arange(12, dtype=np.float64)
    Z, Y, X = np.meshgrid(base, base, base, indexing="ij")
    b = random_hydro_block(rng)
    b[0] = 1e-6 * 4.0 ** (X + Y + Z)
    blocks.append(b)
    dx = 1.0 / 64
    for i, U in enumerate(blocks):
        U = np.ascontiguousarray(U)
        Q = np.empty((5, 26, 10, 10, 10))
        compiled.reconstruct_kernel(U, 1e-12, 1, DIRECTIONS_F, Q)
        FX, FY, FZ = np.empty((5, 8, 8, 9)), np.empty((5, 8, 9, 8)), np.empty((5, 9, 8, 8))
        smax, code, cell = compiled.flux_kernel(Q, 1.4, 1, DIR_PLUS, DIR_MINUS, SIMPSON_W, FX, FY, FZ)
        Uu = U.copy()
        dt = 0.4 * dx / (3.0 * smax) if smax > 0 else 1e-6
        compiled.hydro_update_kernel(Uu, FX, FY, FZ, dt / dx)
        ws = compiled.max_wavespeed_kernel(U, 1.4, 1e-12)
        out[f"U{i}"] = U
        out[f"Qdigest{i}"] = np.array(digest(Q))
        out[f"Qsample{i}"] = Q[:, :, 4, 4, :].copy()
        out[f"FX{i}"], out[f"FY{i}"], out[f"FZ{i}"] = FX, FY, FZ
        out[f"flux_meta{i}"] = np.array([smax, code, cell, dt, ws])
        out[f"Uupd{i}"] = Uu[:, 2:10, 2:10, 2:10].copy()
    # flux error cases on block 0's Q (kernel-level codes, first error)
    U = out["U0"]
    Q = np.empty((5, 26, 10, 10, 10))
    compiled.reconstruct_kernel(U, 1e-12, 1, DIRECTIONS_F, Q)
    errs = []
    for case in range(4):
        Qe = Q.copy()
        if case == 0:
            Qe[0, :, 4, 4, 4] = -1.0
        elif case == 1:
            Qe[4, :, 4, 4, 4] = 1e-9
            Qe[1, :, 4, 4, 4] = 1.0
        elif case == 2:  # both kinds: density later in loop order than pressure
            Qe[0, :, 7, 7, 7] = 0.0
            Qe[4, :, 2, 3, 4] = 1e-12
            Qe[1, :, 2, 3, 4] = 5.0
        else:  # NaN poison must not raise
            Qe[0, :, 5, 5, 5] = np.nan
        FX, FY, FZ = np.empty((5, 8, 8, 9)), np.empty((5, 8, 9, 8)), np.empty((5, 9, 8, 8))
        smax, code, cell = compiled.flux_kernel(Qe, 1.4, 1, DIR_PLUS, DIR_MINUS, SIMPSON_W, FX, FY, FZ)
        errs.append([smax, code, cell])
    out["flux_errors"] = np.array(errs)
    np.savez_compressed(HERE / "hydro_random.npz", **out)


def run_reference_steps(level, state, steps, h, gcfg, gravity):
    """driver.run_scenario's loop (driver.py:162-174) with the reference's
    kernels; gravity evaluated once per step ('every') or only on the final
    step ('last') -- the 6 per-step iterations are identical and never feed
    the hydro."""
    tree = tree_from_global(level, state)
    dts = []
    step_digests = []
    grav_digests = {}
    for step in range(steps):
        if gravity == "every" or (gravity == "last" and step == steps - 1):
            for leaf in tree.leaves:
                leaf.interior("mass")[...] = leaf.interior("rho") * leaf.dx**3
            exchange_ghosts(tree, "gravity")

            def gjob(i):
                t = tree.leaves[i]
                src = neighborhood27(tree, i)
                K.monopole_kernel(t, src, gcfg, "scalar")
                K.multipole_kernel(t, src, gcfg, "scalar")

            list(POOL.map(gjob, range(len(tree.leaves))))
            g = np.stack([global_from_tree(tree, nm) for nm in ("phi", "gx", "gy", "gz")])
            grav_digests[str(step)] = digest(g)
        s_pre = max(K.max_wavespeed(leaf, h) for leaf in tree.leaves)
        dt = h.cfl * tree.dx / (3.0 * s_pre)
        dts.append(fhex(dt))
        for _ in range(3):
            exchange_ghosts(tree, "hydro")

            def hjob(i):
                leaf = tree.leaves[i]
                q = K.reconstruct(leaf, h, "scalar")
                fl = K.flux(leaf, q, h, "scalar")
                K.hydro_update(leaf, fl, dt, h)

            list(POOL.map(hjob, range(len(tree.leaves))))
        U = np.stack([global_from_tree(tree, nm) for nm in FIELDS])
        step_digests.append(digest(U))
        print(f"    step {step} done", flush=True)
    final = {nm: global_from_tree(tree, nm) for nm in FIELDS}
    return final, dts, step_digests, grav_digests


def cfg5(man, level, gravity):
    st = scenarios.config5_state(level)
    h = K.HydroConfig(gamma=1.4)
    gcfg = K.GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    t0 = time.time()
    final, dts, sd, gd = run_reference_steps(level, st, 10, h, gcfg, gravity)
    print(f"  cfg5 L{level}: {time.time() - t0:.1f}s", flush=True)
    man[f"cfg5_L{level}"] = {
        "level": level, "steps": 10, "gravity": gravity, "gamma": fhex(1.4),
        "floor": fhex(scenarios.CONFIG5_FLOOR), "omega": fhex(scenarios.CONFIG5_OMEGA),
        "input_digest": digest(np.stack([st[k] for k in FIELDS])),
        "dts": dts, "step_digests": sd, "gravity_digests": gd,
        "final_field_digests": {k: digest(v) for k, v in final.items()},
    }


def scenario_runs(man):
    """The reference's own driver.run_scenario (driver.py:91-189) end to end:
    fields_bytes-style digests of the final tree (tests/util.py:66-67)."""
    from simdgrid.driver import run_scenario
    from simdgrid.scenarios import ScenarioConfig, init_scenario
    names = ("rho", "sx", "sy", "sz", "E", "phi", "gx", "gy", "gz")
    rec = {}
    for name, level, steps in (("rotating-star-proxy", 1, 2), ("blast", 1, 3), ("rotating-star-proxy", 2, 1)):
        cfg = ScenarioConfig(name, max_level=level, stop_step=steps)
        init = init_scenario(cfg)
        res = run_scenario(cfg, backend="scalar", threads=os.cpu_count() or 4)
        fb = b"".join(leaf.interior(n).tobytes() for leaf in res.tree.leaves for n in names)
        rec[f"{name}_L{level}_s{steps}"] = {
            "level": level, "steps": steps,
            "input_digests": {n: digest(global_from_tree(init, n)) for n in FIELDS + ("mass",)},
            "fields_bytes_sha256": hashlib.sha256(fb).hexdigest(),
            "field_digests": {n: digest(global_from_tree(res.tree, n)) for n in names + ("mass",)},
            "counts": {r.name: r.count for r in res.records},
        }
    man["scenarios"] = rec


def legacy(man):
    """Reference legacy straight-line kernels (kernels/legacy.py): per random
    block Q and fluxes, error cases, and whole legacy-hydro scenario runs."""
    from simdgrid.driver import run_scenario
    from simdgrid.kernels import legacy as LG
    from simdgrid.octree import SubGrid
    from simdgrid.scenarios import ScenarioConfig
    g = np.load(HERE / "hydro_random.npz")
    out = {}
    h = K.HydroConfig()
    for i in range(6):
        sub = SubGrid.allocate(0, (0, 0, 0), 1.0 / 64)
        for v, name in enumerate(FIELDS):
            sub.fields[name][...] = g[f"U{i}"][v]
        q = LG.legacy_reconstruct(sub, h)
        out[f"Qdigest{i}"] = np.array(digest(q.values))
        try:
            fl = LG.legacy_flux(sub, q, h)
            out[f"FX{i}"], out[f"FY{i}"], out[f"FZ{i}"] = fl.fx, fl.fy, fl.fz
            out[f"smax{i}"] = np.array(fl.max_speed)
        except K.KernelError as exc:
            out[f"err{i}"] = np.array(str(exc))
    # kernel-level error codes (first error, left cell) on block 0's Q
    from simdgrid.kernels.geometry import DIR_MINUS, DIR_PLUS, DIRECTIONS_F, SIMPSON_W
    Q = np.empty((5, 26, 10, 10, 10))
    compiled.reconstruct_kernel(np.ascontiguousarray(g["U0"]), 1e-12, 1, DIRECTIONS_F, Q)
    errs = []
    for case in range(4):
        Qe = Q.copy()
        if case == 0:
            Qe[0, :, 4, 4, 4] = -1.0
        elif case == 1:
            Qe[4, :, 4, 4, 4] = 1e-9
            Qe[1, :, 4, 4, 4] = 1.0
        elif case == 2:
            Qe[0, :, 7, 7, 7] = 0.0
            Qe[4, :, 2, 3, 4] = 1e-12
            Qe[1, :, 2, 3, 4] = 5.0
        else:
            Qe[0, :, 5, 5, 5] = np.nan
        FX, FY, FZ = np.empty((5, 8, 8, 9)), np.empty((5, 8, 9, 8)), np.empty((5, 9, 8, 8))
        smax, code, cell = LG._legacy_flux_impl(Qe, 1.4, DIR_PLUS, DIR_MINUS, SIMPSON_W, FX, FY, FZ)
        errs.append([smax, code, cell])
        out[f"errFX{case}"] = FX
    out["flux_errors"] = np.array(errs)
    np.savez_compressed(HERE / "legacy.npz", **out)
    names = ("rho", "sx", "sy", "sz", "E", "phi", "gx", "gy", "gz")
    rec = {}
    for name, level, steps in (("blast", 1, 2), ("rotating-star-proxy", 1, 1)):
        cfg = ScenarioConfig(name, max_level=level, stop_step=steps)
        res = run_scenario(cfg, backend="scalar", threads=os.cpu_count() or 4, hydro_kernel="legacy")
        rec[f"{name}_L{level}_s{steps}"] = {
            "level": level, "steps": steps,
            "field_digests": {n: digest(global_from_tree(res.tree, n)) for n in names},
        }
    man["legacy_scenarios"] = rec


def error_runs(man):
    """The reference's run_scenario (driver.py:91-189, blast: no gravity, 3
    hydro iterations per step) on config-5 level-2 states with NaN cells
    (scenarios.ERROR_CASES): the KernelError message it raises -- the first
    failing hydro iteration's first failing leaf, "step N: ..." (driver.py:83-88)."""
    import simdgrid.driver as RD
    from simdgrid.scenarios import ScenarioConfig
    rec = {}
    for case in scenarios.ERROR_CASES:
        st = scenarios.config5_error_state(case, 2)
        tree = tree_from_global(2, st)
        orig = RD.init_scenario
        RD.init_scenario = lambda cfg, _t=tree: _t
        try:
            RD.run_scenario(ScenarioConfig("blast", max_level=2, stop_step=2), backend="scalar",
                            threads=os.cpu_count() or 4)
            msg = None
        except K.KernelError as exc:
            msg = str(exc)
        finally:
            RD.init_scenario = orig
        rec[case] = {"level": 2, "steps": 2, "gamma": fhex(1.4),
                     "input_digest": digest(np.stack([st[k] for k in FIELDS])), "message": msg}
        print(f"    {case}: {msg}", flush=True)
    man["errors"] = rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-l4", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    man_path = HERE / "manifest.json"
    man = json.loads(man_path.read_text()) if man_path.exists() else {}
    todo = args.only.split(",") if args.only else [
        "cfg1", "tree", "hydro_random", "cfg2", "cfg4", "cfg3", "cfg5_L0", "cfg5_L1", "cfg5_L2", "cfg5_L4",
        "scenarios", "legacy", "errors"]
    for name in todo:
        if name == "cfg5_L4" and args.skip_l4:
            continue
        t0 = time.time()
        print(f"[golden] {name}", flush=True)
        {"cfg1": lambda: gravity_cfg1(), "tree": lambda: gravity_tree(),
         "hydro_random": lambda: hydro_random(), "cfg2": lambda: cfg2_p2p(man),
         "cfg3": lambda: cfg3_m2l(man), "cfg4": lambda: cfg4_hydro(man),
         "cfg5_L0": lambda: cfg5(man, 0, "every"), "cfg5_L1": lambda: cfg5(man, 1, "every"),
         "cfg5_L2": lambda: cfg5(man, 2, "every"), "cfg5_L4": lambda: cfg5(man, 4, "last"),
         "scenarios": lambda: scenario_runs(man), "legacy": lambda: legacy(man),
         "errors": lambda: error_runs(man)}[name]()
        man["_generator"] = "tests/golden/make_golden.py (reference simdgrid, numba compiled path)"
        man_path.write_text(json.dumps(man, indent=1, sort_keys=True))
        print(f"[golden] {name} done in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()

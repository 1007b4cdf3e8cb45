"""Per-kernel device timings (CUDA events, median of reps) on the config-5
state at level L (default 4): gravity kernels (precision exact|fma) and
both hydro paths.  Usage: time_kernels.py [L] [reps] [precision]"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prec = sys.argv[3] if len(sys.argv) > 3 else "exact"
u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
u.load(scenarios.config5_state(level))
u.set_mass()
u._halo(u.mass, 1, u.mv)
u._halo(u.U, 5, u.uv)
B.cluster_aggregate(u.mass, u.dx, u.clusters)


def t(fn):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts[1:])


res = {
    "fill_U": t(lambda: B.fill_periodic(u.U, 5, u.uv, 7)),
    "fill_mass": t(lambda: B.fill_periodic(u.mass, 1, u.mv, 7)),
    "cluster_aggregate": t(lambda: B.cluster_aggregate(u.mass, u.dx, u.clusters)),
    "p2p": t(lambda: B.p2p(u.mass, u.mv, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, u.halo, u.grav, u.gv,
                           precision=prec)),
    "m2l": t(lambda: B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, 1, u.grav, u.gv,
                           precision=prec)),
    "reconstruct": t(lambda: B.reconstruct(u.U, u.uv, u.leaves, u.nleaves, 1e-12, u.Q)),
    "flux": t(lambda: B.flux(u.Q, u.nleaves, 1.4, u.FX, u.FY, u.FZ, u.smax, u.flux_err)),
    "flux_legacy": t(lambda: B.flux_legacy(u.Q, u.nleaves, 1.4, u.FX, u.FY, u.FZ, u.smax, u.flux_err)),
    "hydro_fused": t(lambda: B.hydro_fused(u.U, u.uv, u.leaves, u.nleaves, 1e-12, 1.4, u.FX, u.FY, u.FZ, u.smax,
                                           u.flux_err)),
    "max_wavespeed": t(lambda: B.max_wavespeed(u.U, u.uv, u.leaves, u.nleaves, 1.4, 1e-12, u.ws)),
}
st = torch.empty(u.nleaves, dtype=torch.int32, device=u.U.device)
res["hydro_update"] = t(lambda: B.hydro_update(u.U, u.uv, u.leaves, u.nleaves, u.FX, u.FY, u.FZ, None, None, 1e-9,
                                               u.dx, 0.4, st))
print(json.dumps({k: round(v, 4) for k, v in res.items()}))

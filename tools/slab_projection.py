"""Per-rank device time of one config-5 timestep for a z-slab of 1/P of the
domain (P = 1, 2, 4, 8), kernels only: the compute part of a P-GPU step.
Halos are filled by a local periodic wrap (the NCCL exchange is not timed)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402
from paper_2210_06439_b200.slab import Slab  # noqa: E402

level = 4
prec = sys.argv[1] if len(sys.argv) > 1 else "exact"
st = scenarios.config5_state(level)
res = {}
for P in (1, 2, 4, 8):
    u = grid.UnigridState(level, HydroConfig(gamma=1.4), GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                          slab=Slab(level, 0, P), precision=prec)
    u.load(st)

    def step():
        u.set_mass()
        for _ in range(6):
            B.fill_periodic(u.mass, 1, u.mv, 7)   # stands in for fill(x,y) + z-halo exchange
            u.gravity_kernels()
        u.wavespeed_local()
        B.dt_from_smax(u.s_pre, u.h.cfl, u.dx, u.dt)
        for _ in range(3):
            B.fill_periodic(u.U, 5, u.uv, 7)
            u.hydro_kernels()
    for _ in range(2):
        step()
    u.load(st)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(5):
        step()
    b.record()
    torch.cuda.synchronize()
    res[P] = a.elapsed_time(b) / 5
out = {"precision": prec, "ms_per_step_per_rank": res,
       "projected_strong_scaling_efficiency": {P: res[1] / (P * res[P]) for P in res}}
print(json.dumps(out))

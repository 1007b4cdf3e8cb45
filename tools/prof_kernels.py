"""Small driver for ncu captures: one level-3 (512-subgrid) config-3 gravity
iteration and one config-4 hydro iteration, each run twice (warm-up + the
captured launch).  Usage: python tools/prof_kernels.py [gravity|hydro|all]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
level = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prec = sys.argv[3] if len(sys.argv) > 3 else "exact"
if what in ("gravity", "all"):
    u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                          precision=prec)
    rho = scenarios.polytrope_rho(level, 1e-10)
    z = torch.zeros_like(torch.from_numpy(rho))
    u.load({"rho": rho, "sx": z.numpy(), "sy": z.numpy(), "sz": z.numpy(), "E": rho})
    u.set_mass()
    for _ in range(2):
        u.gravity_iteration()
if what in ("hydro", "all"):
    u = grid.UnigridState(level, HydroConfig(gamma=5.0 / 3.0))
    u.load(scenarios.config4_state(level))
    u.dt.fill_(1e-6)
    for fused in (True, False):
        u.fused_hydro = fused
        for _ in range(2):
            u.hydro_iteration()
torch.cuda.synchronize()
print("ok")

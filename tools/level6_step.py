"""One full timestep at level 6 (512^3 cells, 262,144 subgrids) on one GPU:
resident-memory and 64-bit-indexing check.  Smooth synthetic state (not
config 5's generator, which is scalar-libm and slow at this size); checks
no kernel errors, exact mass conservation (fluxes telescope: periodic), and
prints the step time and peak memory."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_06439_b200 import grid  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
n = 8 << level
x = (np.arange(n) + 0.5) / n
rho = (1.0 + 0.2 * np.sin(2 * np.pi * x)[:, None, None] * np.cos(2 * np.pi * x)[None, :, None]
       + 0.1 * np.sin(4 * np.pi * x)[None, None, :])
st = {"rho": rho, "sx": 0.05 * rho, "sy": np.zeros_like(rho), "sz": -0.03 * rho, "E": 2.5 + 0.0 * rho}
u = grid.UnigridState(level, HydroConfig(gamma=1.4), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
u.load(st)
del st
torch.cuda.synchronize()
m0 = float(u.U[0, 2:-2, 2:-2, 2:-2].sum())
t0 = time.time()
u.step()
torch.cuda.synchronize()
dt = time.time() - t0
u.check_errors()
m1 = float(u.U[0, 2:-2, 2:-2, 2:-2].sum())
g = u.grav
print(json.dumps({"level": level, "subgrids": u.nleaves, "step_s": round(dt, 3),
                  "mass_rel_change": (m1 - m0) / m0, "gravity_finite": bool(torch.isfinite(g).all().item()),
                  "phi_range": [float(g[0].min()), float(g[0].max())],
                  "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 1e9, 1)}))

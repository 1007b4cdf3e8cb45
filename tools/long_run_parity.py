"""Long-horizon parity: N config-5 steps at level L on the GPU (batched
path, exact mode) vs the CPU oracle's step loop (bit-pinned to the
reference by tests/test_oracle_golden.py): every step's dt and the final
state + gravity, bitwise.  Usage: long_run_parity.py [L] [steps]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 4
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
st = scenarios.config5_state(level)
t0 = time.time()
gpu, gdts = grid.run_steps(st, level, steps, hydro=HydroConfig(gamma=1.4),
                           gravity=GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
t_gpu = time.time() - t0
O.use_native()
t0 = time.time()
final, grav, odts = O.run_steps(st, level, steps, gamma=1.4, floor=1e-12, gravity="last")
t_cpu = time.time() - t0
ok_dt = [a == b for a, b in zip(gdts, odts)]
ok_state = {k: bool(np.array_equal(np.ascontiguousarray(gpu[k]).view(np.uint64),
                                   np.ascontiguousarray(final[k]).view(np.uint64))) for k in final}
n = 8 << level
g = np.zeros((4, n, n, n))
for i, (cx, cy, cz) in enumerate(O.leaf_coords(level)):
    g[:, cz * 8:cz * 8 + 8, cy * 8:cy * 8 + 8, cx * 8:cx * 8 + 8] = grav[i].reshape(4, 8, 8, 8)
ok_grav = {k: bool(np.array_equal(gpu[k].view(np.uint64), g[c].view(np.uint64)))
           for c, k in enumerate(("phi", "gx", "gy", "gz"))}
mass0 = float(np.sum(st["rho"]))
mass1 = float(np.sum(gpu["rho"]))
print(json.dumps({"level": level, "steps": steps, "all_dt_bitwise": all(ok_dt), "dt_first_last": [gdts[0], gdts[-1]],
                  "state_bitwise": ok_state, "gravity_bitwise": ok_grav, "gpu_wall_s": round(t_gpu, 2),
                  "oracle_wall_s": round(t_cpu, 2), "total_mass_rel_change": (mass1 - mass0) / mass0}))

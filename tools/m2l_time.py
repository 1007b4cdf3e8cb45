"""Time the batched M2L on the config-5 state at level L (CUDA events,
median of reps) and print a digest of its output -- run twice with and
without SG_M2L_ONE_TARGET=1 for a bit-identity A/B.  Usage: m2l_time.py [L] [reps] [order]"""
import hashlib
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
order = int(sys.argv[3]) if len(sys.argv) > 3 else 1
u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=order))
u.load(scenarios.config5_state(level))
u.set_mass()
u._halo(u.mass, 1, u.mv)
B.cluster_aggregate(u.mass, u.dx, u.clusters)
ts = []
for _ in range(reps + 1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, order, u.grav, u.gv)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
dig = hashlib.sha256(u.grav.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps({"level": level, "order": order, "one_target": os.environ.get("SG_M2L_ONE_TARGET", "0"),
                  "ms": round(statistics.median(ts[1:]), 4), "min_ms": round(min(ts[1:]), 4), "digest": dig}))

"""Time the batched P2P on the config-5 state at level L (CUDA events with
the GPU kept busy, trimmed mean) for the exact and FMA modes and print an
output digest -- run under SG_P2P_ZS=1/2/4 for a bit-identity A/B of the
z-split work units.  Usage: p2p_time.py [L] [reps]"""
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

level = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
u.load(scenarios.config5_state(level))
u.set_mass()
u._halo(u.mass, 1, u.mv)
res = {"level": level, "zs": os.environ.get("SG_P2P_ZS", "auto")}
for prec in ("exact", "fma"):
    ts = []
    for _ in range(reps + 2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100000)
        a.record()
        B.p2p(u.mass, u.mv, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, u.halo, u.grav, u.gv, precision=prec)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = sorted(ts[2:])[reps // 10:reps - reps // 10]
    res[prec + "_us"] = round(statistics.mean(ts), 2)
    res[prec + "_digest"] = hashlib.sha256(u.grav.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps(res))

"""M2L device time (host launch cost hidden) vs batch size on the level-3 config-3 grid: shows the
latency-mode / persistent-kernel crossover.  CUDA event timestamps on the B200 boxes tick every
1.024 us, so each batch size reports the 10%-trimmed mean of 40 reps (the busy-GPU sleep before
each rep dithers the phase), not a median of quantised values."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "exact"
u = grid.UnigridState(3, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
rho = torch.from_numpy(scenarios.config3_rho(3)).cuda()
u.mass[8:-8, 8:-8, 8:-8] = rho * u.dx ** 3
u._halo(u.mass, 1, u.mv)
B.cluster_aggregate(u.mass, u.dx, u.clusters)
res = {}
for n in (1, 2, 3, 4, 6, 8, 12, 16, 32):
    ts = []
    for _ in range(42):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200000)  # keep the GPU busy so host launch cost is not timed
        a.record()
        B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, n, u.dx, u.rad2, u.eps2, 1, u.grav, u.gv, precision=prec)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = sorted(ts[2:])[4:-4]
    res[n] = round(statistics.mean(ts), 2)
print(json.dumps({"precision": prec, "m2l_us_by_batch": res}))

"""Config-1 single-subgrid M2L (cluster_aggregate + m2l) timed with CUDA events
(GPU kept busy before each rep so host launch cost is hidden, and without);
used for ncu captures of the latency path."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import scenarios  # noqa: E402
from paper_2210_06439_b200.batched import View  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40  # events tick at 1.024 us: trimmed mean
cube = torch.from_numpy(scenarios.config1_cube(0)).cuda()
cl = torch.empty((12, 12, 12, 4), dtype=torch.float64, device="cuda")
res = torch.empty((4, 8, 8, 8), dtype=torch.float64, device="cuda")
dx = 1.0 / 64
rad = dx / 0.34
eps = 0.5 * dx


def c1():
    B.cluster_aggregate(cube, dx, cl)
    B.m2l(cube, View(8, 8, 8, 8), cl, 0, None, 1, dx, rad * rad, eps * eps, 1, res, View(8, 8, 8, 0))


out = {}
for busy in (True, False):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if busy:
            torch.cuda._sleep(200000)
        a.record()
        c1()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts = sorted(ts[1:])[reps // 10:reps - reps // 10]
    out["busy" if busy else "idle"] = round(statistics.mean(ts), 2)
print(json.dumps({"config1_us": out}))

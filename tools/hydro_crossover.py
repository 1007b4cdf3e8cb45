"""Fused vs unfused (reconstruct + flux) hydro iteration time vs batch size:
z-slabs of the level-4 config-5 grid with 4096/P subgrids (P = 1, 2, 4, 8,
16), CUDA-event medians, host enqueue hidden."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200.kernels import HydroConfig  # noqa: E402
from paper_2210_06439_b200.slab import Slab  # noqa: E402

st = scenarios.config5_state(4)
res = {}
for P in (1, 2, 4, 8, 16):
    u = grid.UnigridState(4, HydroConfig(gamma=1.4), slab=Slab(4, 0, P))
    u.load(st)
    u.dt.fill_(1e-7)
    out = {}
    for fused in (True, False):
        u.fused_hydro = fused
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(200000)
            a.record()
            u.hydro_kernels()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out["fused" if fused else "unfused"] = round(statistics.median(ts[2:]), 4)
    res[u.nleaves] = out
print(json.dumps({"hydro_iteration_ms_by_subgrids": res}))

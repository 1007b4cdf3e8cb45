import json, statistics, sys
from pathlib import Path
sys.path.insert(0, "/root/repo")
import torch
from paper_2210_06439_b200 import batched as B
from paper_2210_06439_b200 import grid, scenarios
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig
u = grid.UnigridState(3, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
rho = torch.from_numpy(scenarios.config3_rho(3)).cuda()
u.mass[8:-8, 8:-8, 8:-8] = rho * u.dx ** 3
u._halo(u.mass, 1, u.mv)
B.cluster_aggregate(u.mass, u.dx, u.clusters)
ws = B.m2l_workspace(1)
def call():
    B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, 1, u.dx, u.rad2, u.eps2, 1, u.grav, u.gv, workspace=ws)
for sl in (200000, 2000000):
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(sl); a.record(); call(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    print("sleep", sl, "single", round(statistics.median(ts[2:]), 2))
for n in (10, 50):
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2000000); a.record()
        for _ in range(n): call()
        b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / n)
    print("back-to-back", n, "per call", round(statistics.median(ts[2:]), 2))
# graph of 10 calls
s = torch.cuda.Stream()

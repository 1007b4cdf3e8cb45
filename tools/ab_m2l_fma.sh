#!/bin/bash
cp paper_2210_06439_b200/libsg.so /tmp/libsg_orig.so
for f in paper_2210_06439_b200/libsg_*.so; do
  cp $f paper_2210_06439_b200/libsg.so
  python - "$f" <<'PY'
import sys; sys.path.insert(0, ".")
import torch, statistics
from paper_2210_06439_b200 import batched as B, grid, scenarios
from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig
u = grid.UnigridState(4, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
u.load(scenarios.config5_state(4)); u.set_mass(); u._halo(u.mass, 1, u.mv); B.cluster_aggregate(u.mass, u.dx, u.clusters)
res = {}
for prec in ("exact", "fma"):
    ts = []
    for r in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True); a.record()
        B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, 1, u.grav, u.gv, precision=prec)
        b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res[prec] = round(statistics.median(ts[1:]), 4)
print(sys.argv[1], res)
PY
done
cp /tmp/libsg_orig.so paper_2210_06439_b200/libsg.so

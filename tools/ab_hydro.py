"""Fused hydro A/B at level L (default 4) on the config-5 state: times the
default (deduplicated) kernel and, with SG_HYDRO_FUSED=rebuild, the round-1
kernel; checks the two are bit-identical.  Usage: ab_hydro.py [L] [reps]"""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
if os.environ.get("_AB_CHILD"):
    sys.path.insert(0, str(REPO))
    import numpy as np
    import torch
    from paper_2210_06439_b200 import batched as B
    from paper_2210_06439_b200 import grid, scenarios
    from paper_2210_06439_b200.kernels import GravityConfig, HydroConfig
    level, reps = int(sys.argv[1]), int(sys.argv[2])
    u = grid.UnigridState(level, HydroConfig(), GravityConfig(theta=0.34, eps=0.5, expansion_order=1))
    u.load(scenarios.config5_state(level))
    u._halo(u.U, 5, u.uv)
    fn = lambda: B.hydro_fused(u.U, u.uv, u.leaves, u.nleaves, 1e-12, 1.4, u.FX, u.FY, u.FZ, u.smax,  # noqa
                               u.flux_err)
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out = np.concatenate([x.cpu().numpy().ravel() for x in (u.FX, u.FY, u.FZ, u.smax)])
    np.save(sys.argv[3], out)
    np.save(sys.argv[3] + ".err.npy", u.flux_err.cpu().numpy())
    print(json.dumps({"ms": statistics.median(ts[1:]), "all": ts[1:]}))
    sys.exit(0)
level = sys.argv[1] if len(sys.argv) > 1 else "4"
reps = sys.argv[2] if len(sys.argv) > 2 else "10"
res = {}
for name, env in (("dedup", {}), ("rebuild", {"SG_HYDRO_FUSED": "rebuild"})):
    e = dict(os.environ, _AB_CHILD="1", **env)
    r = subprocess.run([sys.executable, __file__, level, reps, f"/tmp/ab_{name}.npy"], env=e, capture_output=True,
                       text=True)
    if r.returncode:
        print(r.stderr)
        sys.exit(1)
    res[name] = json.loads(r.stdout.strip().splitlines()[-1])["ms"]
import numpy as np  # noqa: E402
a, b = np.load("/tmp/ab_dedup.npy"), np.load("/tmp/ab_rebuild.npy")
same = a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
same_err = np.array_equal(np.load("/tmp/ab_dedup.npy.err.npy"), np.load("/tmp/ab_rebuild.npy.err.npy"))
print(json.dumps({"level": int(level), "ms": res, "bit_identical": bool(same), "err_identical": bool(same_err)}))

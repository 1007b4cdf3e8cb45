"""Small cases covering every kernel for compute-sanitizer runs: level-1
gravity + hydro (fused, unfused, legacy), the drop-in per-subgrid paths
(single-leaf M2L split over 16 CTAs, P2P param + smem stencils), gather,
a 2-slab local exchange step, and level-3 gravity + hydro iterations in
both precisions (persistent M2L, FMA mirror M2L, 8-target P2P)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2210_06439_b200 import driver as D  # noqa: E402
from paper_2210_06439_b200 import grid, scenarios  # noqa: E402
from paper_2210_06439_b200 import kernels as K  # noqa: E402
from paper_2210_06439_b200.octree import neighborhood27  # noqa: E402

for hk in ("cuda", "legacy"):
    D.run_scenario(D.ScenarioConfig("rotating-star-proxy", max_level=1, stop_step=1), hydro_kernel=hk)
tree = D.init_scenario(D.ScenarioConfig("rotating-star-proxy", max_level=1, stop_step=1))
for theta in (0.34, 0.2):
    K.monopole_kernel(tree.leaves[2], neighborhood27(tree, 2), K.GravityConfig(theta=theta))
    K.multipole_kernel(tree.leaves[5], neighborhood27(tree, 5), K.GravityConfig(theta=theta, expansion_order=1))
st = grid.UnigridState.from_tree(tree)
st.set_mass()
st.source_cubes("mass", 8)
st.source_cubes("rho", 2)
ls = grid.LocalSlabs(1, 2)
ls.load(scenarios.config5_state(1))
ls.step()
ls.check_errors()
# persistent M2L (>= 148 subgrids), the FMA mirror kernel and the 8-target P2P
for prec in ("exact", "fma"):
    u = grid.UnigridState(3, K.HydroConfig(), K.GravityConfig(theta=0.34, eps=0.5, expansion_order=1), precision=prec)
    u.load(scenarios.config5_state(3))
    u.set_mass()
    u.gravity_iteration()
    u.wavespeed_dt()
    u.hydro_iteration()
    u.check_errors()
torch.cuda.synchronize()
print("sanitize cases done")
print("sanitize cases ok")

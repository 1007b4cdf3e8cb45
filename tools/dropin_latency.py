"""Per-call wall-clock cost of the drop-in entry points (kernels.py, the
reference's per-subgrid API) on one subgrid of a level-1 tree: host gather,
H2D, kernels, D2H and the write-back into SubGrid.fields, median of reps --
next to the same kernel on one host core through the C oracle (the
reference's compiled per-subgrid kernel, restated)."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2210_06439_b200 import kernels as K  # noqa: E402
from paper_2210_06439_b200 import octree  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(0)
tree = octree.build_unigrid(1)
for name in ("mass",):
    octree.set_global_field(tree, name, rng.random((16, 16, 16)) * (1 / 16) ** 3)
for leaf in tree.leaves:
    leaf.fields["rho"][...] = 1.0 + 0.1 * rng.random((12, 12, 12))
    for n in ("sx", "sy", "sz"):
        leaf.fields[n][...] = 0.01 * rng.standard_normal((12, 12, 12))
    leaf.fields["E"][...] = 2.5 + 0.1 * rng.random((12, 12, 12))
leaf, nb = tree.leaves[0], octree.neighborhood27(tree, 0)
g = K.GravityConfig(theta=0.34, expansion_order=1)
h = K.HydroConfig()


def wall(fn, n=reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


q = K.reconstruct(leaf, h)
fl = K.flux(leaf, q, h)
res = {
    "monopole_kernel": wall(lambda: K.monopole_kernel(leaf, nb, g)),
    "multipole_kernel": wall(lambda: K.multipole_kernel(leaf, nb, g)),
    "reconstruct": wall(lambda: K.reconstruct(leaf, h)),
    "flux": wall(lambda: K.flux(leaf, q, h)),
    "max_wavespeed": wall(lambda: K.max_wavespeed(leaf, h)),
}
# one host core, C oracle, same subgrid
O.build()
cube8 = octree.source_cube(nb, "mass", 8)
cube2 = octree.source_cube(nb, "mass", 2)
U = np.stack([leaf.fields[n] for n in ("rho", "sx", "sy", "sz", "E")])
Q = O.reconstruct(U, h.positivity_floor)
cpu = {
    "monopole_kernel": wall(lambda: O.monopole(cube2, leaf.dx, 0.34, 0.5), 3),
    "multipole_kernel": wall(lambda: O.multipole(cube8, leaf.dx, 0.34, 0.5, 1), 1),
    "reconstruct": wall(lambda: O.reconstruct(U, h.positivity_floor), 5),
    "flux": wall(lambda: O.flux(Q, h.gamma), 5),
    "max_wavespeed": wall(lambda: O.max_wavespeed(U, h.gamma, h.positivity_floor), 5),
}
print(json.dumps({"dropin_call_us": {k: round(v, 1) for k, v in res.items()},
                  "oracle_1core_us": {k: round(v, 1) for k, v in cpu.items()}}))

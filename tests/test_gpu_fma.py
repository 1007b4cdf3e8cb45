"""precision="fma": the gravity kernels with FMA-contracted, re-associated
far/near terms (north_star: "FP64 CUDA-core FMAs ... match the Python
reference to a relative tolerance of 1e-12 in FP64, per output component").

Tolerance, written here: for every output component array (phi, gx, gy, gz)
max |fma - ref| <= 1e-12 * max |ref| (max-norm relative; elementwise relative
error is meaningless where a component crosses zero).  ``ref`` is the
reference itself (golden arrays) or our exact path, which is bit-identical to
the reference (tests/test_gpu_parity.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import digest, load_npz

pytestmark = pytest.mark.gpu

from paper_2210_06439_b200 import batched as B  # noqa: E402
from paper_2210_06439_b200 import grid as G  # noqa: E402
from paper_2210_06439_b200 import kernels as K  # noqa: E402
from paper_2210_06439_b200 import scenarios  # noqa: E402
from paper_2210_06439_b200.batched import View  # noqa: E402

TOL = 1e-12


def maxnorm_rel(got, want) -> float:
    return float(np.max(np.abs(got - want)) / np.max(np.abs(want)))


def check(got, want):
    for c in range(4):
        err = maxnorm_rel(got[c], want[c])
        assert err <= TOL, (c, err)
    return max(maxnorm_rel(got[c], want[c]) for c in range(4))


@pytest.mark.parametrize("theta,order", [(0.34, 1), (0.34, 0), (0.5, 1), (0.2, 1)])
def test_cfg1_m2l_fma_vs_reference(theta, order):
    g = load_npz("gravity_cfg1.npz")
    dx = 1.0 / 64
    cube = torch.from_numpy(g["cube"]).cuda()
    cl = torch.empty((12, 12, 12, 4), dtype=torch.float64, device="cuda")
    B.cluster_aggregate(cube, dx, cl)
    cfg = K.GravityConfig(theta=theta, eps=0.5, expansion_order=order)
    rad2, eps2 = K.gravity_params(dx, cfg)
    out = torch.zeros((4, 8, 8, 8), dtype=torch.float64, device="cuda")
    B.m2l(cube, View(8, 8, 8, 8), cl, 0, None, 1, dx, rad2, eps2, order, out, View(8, 8, 8, 0), precision="fma")
    key = f"m2l_t{int(theta * 100)}_o{order}"
    if key in g:
        check(out.cpu().numpy(), g[key])
    else:  # theta 0.2 has no cfg1 golden: compare with the exact path
        ref = torch.zeros_like(out)
        B.m2l(cube, View(8, 8, 8, 8), cl, 0, None, 1, dx, rad2, eps2, order, ref, View(8, 8, 8, 0))
        check(out.cpu().numpy(), ref.cpu().numpy())


@pytest.mark.parametrize("kind", ["p2p", "m2l"])
def test_batched_fma_vs_exact_level3(kind):
    level, n = 3, 64
    rho = scenarios.config2_rho(1, level) if kind == "p2p" else scenarios.config3_rho(level)
    z = np.zeros_like(rho)
    outs = {}
    for prec in ("exact", "fma"):
        u = G.UnigridState(level, K.HydroConfig(), K.GravityConfig(theta=0.34, eps=0.5, expansion_order=1),
                           precision=prec)
        u.load({"rho": rho, "sx": z, "sy": z, "sz": z, "E": rho})
        u.set_mass()
        u._halo(u.mass, 1, u.mv)
        B.cluster_aggregate(u.mass, u.dx, u.clusters)
        if kind == "p2p":
            B.p2p(u.mass, u.mv, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, u.halo, u.grav, u.gv, precision=prec)
        else:
            B.m2l(u.mass, u.mv, u.clusters, 0, u.leaves, u.nleaves, u.dx, u.rad2, u.eps2, 1, u.grav, u.gv,
                  precision=prec)
        outs[prec] = u.grav.cpu().numpy()
    assert not np.array_equal(outs["fma"], outs["exact"])  # really a different arithmetic
    check(outs["fma"], outs["exact"])


def test_cfg5_level4_fma_mode(manifest):
    """Ten config-5 steps with FMA gravity: the hydro state is still
    bit-identical to the reference (gravity never feeds the hydro), and the
    final gravity is within the tolerance of the exact path."""
    m = manifest["cfg5_L4"]
    st = scenarios.config5_state(4)
    if digest(np.stack([st[k] for k in ("rho", "sx", "sy", "sz", "E")])) != m["input_digest"]:
        pytest.fail("input generator mismatch: config-5 generator differs on this host -- the golden inputs cannot be reproduced, parity coverage would be lost")
    g = K.GravityConfig(theta=0.34, eps=0.5, expansion_order=1)
    u = G.UnigridState(4, K.HydroConfig(gamma=1.4), g, precision="fma")
    u.load(st)
    for s in range(10):
        u.step()
    u.check_errors()
    out = u.fetch()
    for k in ("rho", "sx", "sy", "sz", "E"):
        assert digest(out[k]) == m["final_field_digests"][k], k
    ref = G.UnigridState(4, K.HydroConfig(gamma=1.4), g)
    ref.U.copy_(u.U)                       # same state -> same mass: compare one gravity pass
    ref.set_mass()
    ref.gravity_iteration()
    u.set_mass()
    u.gravity_iteration()
    check(u.grav.cpu().numpy(), ref.grav.cpu().numpy())

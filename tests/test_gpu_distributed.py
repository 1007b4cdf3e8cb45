"""The multi-rank z-slab step executed for real: P processes,
each a torch.distributed rank owning one z-slab of the config-5 grid, run the
full UnigridState.step -- padded-field halo exchange (grid.py _halo ->
slab.exchange_z_halo), the MAX all-reduce of the pre-step wave speed
(slab.allreduce_max_) and the cross-rank first-error report
(slab.allreduce_min_int + first_error_across_ranks) -- with the CUDA kernels,
and must reproduce the reference goldens bit for bit.

All ranks share the one GPU of the test box, so the collectives run over
gloo with host-staged buffers (slab._host_staged); kernels never wait on
another rank (every exchange completes on the host between launches).  The
NCCL path differs only in the transport of the same buffers.

Also here: first-failing-iteration error semantics (the reference raises
right after the first hydro iteration that fails, driver.py:83-88/173-174)
against messages the reference itself produced (manifest "errors")."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from conftest import digest
from paper_2210_06439_b200 import grid as G
from paper_2210_06439_b200 import kernels as K
from paper_2210_06439_b200 import octree, scenarios

pytestmark = pytest.mark.gpu

GRAV = dict(theta=0.34, eps=0.5, expansion_order=1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, job, q):
    import torch.distributed as dist

    from paper_2210_06439_b200.slab import Slab
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kind, arg = job
        slab = Slab(2, rank, world)
        if kind == "steps":
            m = arg
            u = G.UnigridState(2, K.HydroConfig(gamma=float.fromhex(m["gamma"])), K.GravityConfig(**GRAV),
                               slab=slab)
            u.load(scenarios.config5_state(2))
            for s in range(m["steps"]):
                u.step()
                u.check_errors()
                p = G.U_PAD
                Uc = u.U[:, p:p + u.nz, p:p + u.n, p:p + u.n].cpu().numpy()
                g = u.grav.cpu().numpy() if str(s) in m["gravity_digests"] else None
                q.put((rank, s, u.dt.item(), Uc, g))
            q.put((rank, "done", None, None, None))
        else:  # error case: every rank must raise the same message
            u = G.UnigridState(2, K.HydroConfig(gamma=1.4), K.GravityConfig(**GRAV), slab=slab)
            u.load(scenarios.config5_error_state(arg, 2))
            msg = None
            for _ in range(2):
                u.step(0)
                try:
                    u.check_errors()
                except K.KernelError as exc:
                    msg = str(exc)
                    break
            q.put((rank, msg))
    finally:
        dist.destroy_process_group()


def _spawn(world, job, nmsg):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, job, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        msgs = [q.get(timeout=600) for _ in range(nmsg)]
    finally:
        for p in procs:
            p.join(timeout=120)
    for p in procs:
        assert p.exitcode == 0, f"rank process exited with {p.exitcode}"
    return msgs


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_cfg5_level2_matches_golden(manifest, world):
    """P ranks x one z-slab each, 10 full steps (6 gravity + 3 hydro
    iterations per step): per-step dt, per-step state digests, gravity
    digests and the final fields equal the reference run."""
    m = manifest["cfg5_L2"]
    st = scenarios.config5_state(2)
    if digest(np.stack([st[k] for k in octree.HYDRO_FIELDS])) != m["input_digest"]:
        pytest.fail("input generator mismatch: config-5 generator differs on this host")
    steps = m["steps"]
    msgs = _spawn(world, ("steps", m), world * (steps + 1))
    per = {}
    for rank, s, dt, Uc, g in msgs:
        if s != "done":
            per[(s, rank)] = (dt, Uc, g)
    for s in range(steps):
        dts = {per[(s, r)][0] for r in range(world)}
        assert len(dts) == 1, f"ranks disagree on dt at step {s}"
        assert dts.pop().hex() == m["dts"][s], s
        U = np.concatenate([per[(s, r)][1] for r in range(world)], axis=1)
        assert digest(U) == m["step_digests"][s], f"state differs after step {s}"
        if str(s) in m["gravity_digests"]:
            g = np.concatenate([per[(s, r)][2] for r in range(world)], axis=1)
            assert digest(g) == m["gravity_digests"][str(s)], f"gravity differs at step {s}"
    U = np.concatenate([per[(steps - 1, r)][1] for r in range(world)], axis=1)
    for v, k in enumerate(octree.HYDRO_FIELDS):
        assert digest(U[v]) == m["final_field_digests"][k], k


@pytest.mark.parametrize("case", sorted(scenarios.ERROR_CASES))
def test_distributed_first_error_matches_reference(manifest, case):
    """Two ranks: both raise the reference's message (first failing hydro
    iteration, then first failing leaf in global Morton order)."""
    want = manifest["errors"][case]["message"]
    msgs = _spawn(2, ("error", case), 2)
    assert {m for _, m in msgs} == {want}


@pytest.mark.parametrize("case", sorted(scenarios.ERROR_CASES))
def test_first_failing_iteration_single_and_local_slabs(manifest, case):
    """One slab and 4 in-process slabs: 3 hydro iterations per step run
    before the check, yet the message is the reference's -- errors of
    iterations after the first failing one (here the NaN reaching leaf
    (0, 0, 0) in iteration 2) are not latched."""
    rec = manifest["errors"][case]
    st = scenarios.config5_error_state(case, 2)
    if digest(np.stack([st[k] for k in octree.HYDRO_FIELDS])) != rec["input_digest"]:
        pytest.fail("input generator mismatch for the error case")
    h = K.HydroConfig(gamma=1.4)
    g = K.GravityConfig(**GRAV)
    one = G.UnigridState(2, h, g)
    one.load(st)
    one.step(0)
    assert one.failing_iteration() == 0
    with pytest.raises(K.KernelError) as got:
        one.check_errors()
    assert str(got.value) == rec["message"]
    # the NaN did reach leaf (0, 0, 0) in a later iteration of the same step
    rho = one.fetch()["rho"]
    assert np.isnan(rho[0:8, 0:8, 0:8]).any()
    four = G.LocalSlabs(2, 4, h, g)
    four.load(st)
    four.step(0)
    with pytest.raises(K.KernelError) as got:
        four.check_errors()
    assert str(got.value) == rec["message"]


def test_state_on_non_current_device_rejects_cpu():
    with pytest.raises(ValueError, match="CUDA device"):
        G.UnigridState(1, K.HydroConfig(), K.GravityConfig(**GRAV), device="cpu")

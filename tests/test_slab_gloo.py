"""Multi-process z-slab plumbing on CPU: world_size 2 and 4 over gloo run the
same torch.distributed halo exchange and MAX reduction the NCCL path uses,
and must reproduce the periodic padding of the global field exactly."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2210_06439_b200.slab import Slab, allreduce_max_, allreduce_min_int, exchange_z_halo, first_error_across_ranks


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, level, pad, ncomp, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        slab = Slab(level, rank, world)
        n = slab.n
        g = np.random.default_rng(2).uniform(size=(ncomp, n, n, n))
        want = np.pad(g, ((0, 0), (pad, pad), (pad, pad), (pad, pad)), mode="wrap")
        f = torch.zeros((ncomp, slab.nz + 2 * pad, n + 2 * pad, n + 2 * pad), dtype=torch.float64)
        f[:, pad:pad + slab.nz] = torch.from_numpy(want[:, pad + slab.z0:pad + slab.z0 + slab.nz])
        exchange_z_halo(f, pad, slab)
        ok = np.array_equal(f.numpy(), want[:, slab.z0:slab.z0 + slab.nz + 2 * pad])
        t = torch.tensor([float(rank + 1) * 0.5], dtype=torch.float64)
        allreduce_max_(t, slab)
        # first failing iteration: the minimum over ranks (OPEN on rank 0)
        it = allreduce_min_int(2 ** 31 - 1 if rank == 0 else 5 + rank, slab)
        q.put((rank, ok, t.item(), it))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,level,pad,ncomp", [(2, 2, 8, 1), (2, 2, 2, 5), (4, 2, 8, 1), (4, 2, 2, 5)])
def test_gloo_halo_exchange_matches_periodic_pad(world, level, pad, ncomp):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, level, pad, ncomp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, mx, it in res:
        assert ok, f"rank {rank} halo mismatch"
        assert mx == world * 0.5
        assert it == 6


def _err_worker(rank, world, port, cands, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, first_error_across_ranks(cands[rank], Slab(2, rank, world))))
    finally:
        dist.destroy_process_group()


def test_gloo_first_error_across_ranks():
    """Every rank reports the failing leaf with the smallest Morton key over
    all slabs (rank 1's here), or None when no rank failed."""
    ctx = mp.get_context("spawn")
    for cands, want in (([(27, "leaf (3, 3, 0)"), (4, "leaf (0, 0, 1)"), None, (40, "x")], (4, "leaf (0, 0, 1)")),
                        ([None, None, None, None], None)):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_err_worker, args=(r, 4, port, cands, q)) for r in range(4)]
        for p in procs:
            p.start()
        res = [q.get(timeout=120) for _ in range(4)]
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        for rank, got in res:
            assert (tuple(got) if got is not None else None) == want, rank

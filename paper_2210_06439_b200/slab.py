"""z-slab domain decomposition and halo exchange for the multi-GPU step.

One process per GPU owns ``layers`` consecutive z-layers of subgrids of a
periodic level-L unigrid.  Padded fields are stored per component as
(nz_local + 2p, n + 2p, n + 2p) arrays [z][y][x], so a z-halo is a
contiguous block of whole padded planes: the exchange sends each neighbour
its boundary interior planes directly from the field (no pack kernels) with
``torch.distributed`` point-to-point ops -- NCCL over NVLink on GPUs, gloo on
CPU for the host-logic tests.  x/y pads are filled on-device before the
exchange so the planes travel complete (corners included).

This replaces the in-process ghost copy of the reference
(octree.exchange_ghosts, reference octree.py:149-167; source_cube 186-214):
with P = 1 the z wrap is a local periodic fill instead.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Slab:
    level: int
    rank: int = 0
    world: int = 1

    def __post_init__(self):
        na = 1 << self.level
        if self.world < 1 or na % self.world:
            raise ValueError(f"{na} subgrid layers cannot be split over {self.world} ranks")

    @property
    def n(self) -> int:
        return 8 << self.level

    @property
    def layers(self) -> int:
        return (1 << self.level) // self.world

    @property
    def nz(self) -> int:
        return 8 * self.layers

    @property
    def z0(self) -> int:
        return self.rank * self.nz

    @property
    def up(self) -> int:
        return (self.rank + 1) % self.world

    @property
    def down(self) -> int:
        return (self.rank - 1) % self.world

    def leaf_coords(self) -> torch.Tensor:
        """(cx, cy, cz_local) of this rank's leaves, z-major (int32)."""
        na = 1 << self.level
        c = [(x, y, z) for z in range(self.layers) for y in range(na) for x in range(na)]
        return torch.tensor(c, dtype=torch.int32)

    def global_leaf_coords(self) -> torch.Tensor:
        c = self.leaf_coords().clone()
        c[:, 2] += self.rank * self.layers
        return c


def exchange_z_halo(field: torch.Tensor, pad: int, slab: Slab, group=None) -> None:
    """Fill the z pads of a padded field (ncomp, nz+2p, Y, X) from the
    periodic z-neighbour ranks.  Each rank sends its top `pad` interior
    planes up and its bottom `pad` planes down; matching is by posting order,
    which also makes world == 2 (up == down) correct."""
    if slab.world == 1:
        raise ValueError("single rank: use the local periodic fill")
    nz = slab.nz
    if nz < pad:
        raise ValueError(f"slab of {nz} planes is thinner than the halo ({pad})")
    ncomp = field.shape[0]
    ops = []
    for c in range(ncomp):
        f = field[c]
        top = f[nz:nz + pad]            # interior planes [nz-pad+pad, nz+pad)
        bottom = f[pad:2 * pad]         # interior planes [pad, 2pad)
        lower_pad = f[0:pad]
        upper_pad = f[nz + pad:nz + 2 * pad]
        ops.append(dist.P2POp(dist.isend, top, slab.up, group))
        ops.append(dist.P2POp(dist.isend, bottom, slab.down, group))
        ops.append(dist.P2POp(dist.irecv, lower_pad, slab.down, group))
        ops.append(dist.P2POp(dist.irecv, upper_pad, slab.up, group))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def exchange_z_halo_local(fields: list, pad: int, nz: int) -> None:
    """The same exchange between P slabs held by one process (slab r at
    fields[r], each (ncomp, nz+2p, Y, X)): used to run the z-slab
    decomposition on a single device, e.g. to check P-invariance."""
    P = len(fields)
    if nz < pad:
        raise ValueError(f"slab of {nz} planes is thinner than the halo ({pad})")
    for r, f in enumerate(fields):
        down, up = fields[(r - 1) % P], fields[(r + 1) % P]
        f[:, 0:pad].copy_(down[:, nz:nz + pad])
        f[:, nz + pad:nz + 2 * pad].copy_(up[:, pad:2 * pad])


def allreduce_max_(t: torch.Tensor, slab: Slab, group=None) -> None:
    """dt reduction across ranks: MAX is order-independent, so dt is bitwise
    identical for every P (driver.py:170-171)."""
    if slab.world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)


def first_error_across_ranks(candidate, slab: Slab, group=None):
    """Error reporting across slabs: each rank passes its first failing
    leaf as (Morton key, message) or None; every rank gets back the global
    first one (the reference reports the first failing leaf in leaf_iter
    order, driver.py:83-88, which interleaves z) or None."""
    if slab.world == 1:
        return candidate
    found = [None] * slab.world
    dist.all_gather_object(found, candidate, group=group)
    found = [c for c in found if c is not None]
    return min(found, key=lambda c: c[0]) if found else None

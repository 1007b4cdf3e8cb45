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


def _host_staged(t: torch.Tensor, group) -> bool:
    """CUDA tensors over a non-NCCL backend (gloo: several ranks sharing one
    GPU in the tests) travel through host copies; NCCL sends device memory."""
    return t.is_cuda and dist.get_backend(group) != "nccl"


def exchange_z_halo(field: torch.Tensor, pad: int, slab: Slab, group=None) -> None:
    """Fill the z pads of a padded field (ncomp, nz+2p, Y, X) from the
    periodic z-neighbour ranks.  Each rank sends its top `pad` interior
    planes up and its bottom `pad` planes down; matching is by posting order,
    which also makes world == 2 (up == down) correct.  One message per
    direction: a one-component field sends its contiguous planes in place,
    several components are packed into one buffer (a single device copy), so
    a U exchange is 2 sends + 2 receives, not 4 per component."""
    if slab.world == 1:
        raise ValueError("single rank: use the local periodic fill")
    nz = slab.nz
    if nz < pad:
        raise ValueError(f"slab of {nz} planes is thinner than the halo ({pad})")
    top = field[:, nz:nz + pad]             # interior planes [nz-pad, nz)
    bottom = field[:, pad:2 * pad]          # interior planes [0, pad)
    lower_pad = field[:, 0:pad]
    upper_pad = field[:, nz + pad:nz + 2 * pad]
    staged = _host_staged(field, group)
    direct = field.shape[0] == 1 and not staged
    if direct:
        s_up, s_down, r_low, r_up = top, bottom, lower_pad, upper_pad
    else:
        dev = "cpu" if staged else field.device
        s_up = top.to(dev, copy=True).contiguous()
        s_down = bottom.to(dev, copy=True).contiguous()
        r_low = torch.empty(s_up.shape, dtype=field.dtype, device=dev)
        r_up = torch.empty(s_up.shape, dtype=field.dtype, device=dev)
    ops = [dist.P2POp(dist.isend, s_up, slab.up, group),
           dist.P2POp(dist.isend, s_down, slab.down, group),
           dist.P2POp(dist.irecv, r_low, slab.down, group),
           dist.P2POp(dist.irecv, r_up, slab.up, group)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    if not direct:
        lower_pad.copy_(r_low)
        upper_pad.copy_(r_up)


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
    if slab.world == 1:
        return
    if _host_staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)


def allreduce_min_int(v: int, slab: Slab, group=None) -> int:
    """Global minimum of one integer per rank (the first failing hydro
    iteration; a tensor collective, so the no-error path never pickles)."""
    if slab.world == 1:
        return v
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t.item())


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

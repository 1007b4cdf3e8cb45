"""Device-resident unigrid state and the batched full step.

The reference advances a tree of 8^L SubGrids with one thread-pool task per
leaf per kernel (reference driver.py:91-189): per step, mass = rho*dx^3, then
6 x (ghost exchange + monopole + multipole), then dt from the pre-step max
wave speed, then 3 x (ghost exchange + reconstruct + flux + update).  Here
the same step runs on padded global fields resident in HBM:

  U         (5, nz+4, n+4, n+4)     hydro state, pad 2 (= G ghosts)
  mass      (nz+16, n+16, n+16)     pad 8 (the M2L 24^3 neighbourhood)
  clusters  ((nz+16)/2, (n+16)/2, (n+16)/2, 4)   {M, Dx, Dy, Dz}
  grav      (4, nz, n, n)           phi, gx, gy, gz
  Q         (B, 5, 26, 10^3)        reconstruction (drop-in unfused path)

with one launch per kernel over all B leaves, the ghost exchange replaced by
an on-device periodic fill (plus the NCCL z-slab halo for P > 1, slab.py),
and dt computed on device.  Results are bit-identical to the reference loop.
"""

from __future__ import annotations

import functools
import os

import numpy as np
import torch

from . import batched as B
from .batched import View
from .kernels import GravityConfig, HydroConfig, KernelError, decode_flux_error, gravity_halo, gravity_params
from .octree import HYDRO_FIELDS, morton_key
from .slab import Slab, allreduce_max_, allreduce_min_int, exchange_z_halo, exchange_z_halo_local, \
    first_error_across_ranks

MASS_PAD = 8
U_PAD = 2
GATE_OPEN = 2 ** 31 - 1   # err_gate value while no hydro iteration has failed


def _on_device(fn):
    """Run a UnigridState method with its device current, so every launch
    (batched._stream() = the current device's current stream) and every
    scratch allocation target self.device even when the caller's current
    device differs."""
    @functools.wraps(fn)
    def wrapped(self, *a, **kw):
        with torch.cuda.device(self.device):
            return fn(self, *a, **kw)
    return wrapped


class UnigridState:
    """One rank's z-slab of a periodic level-L unigrid, resident on a GPU."""

    def __init__(self, level: int, hydro: HydroConfig | None = None, gravity: GravityConfig | None = None,
                 slab: Slab | None = None, device=None, group=None, fused_hydro: bool = True,
                 legacy_flux: bool = False, precision: str = "exact"):
        B.require_device()
        self.level = level
        self.slab = slab or Slab(level)
        if self.slab.level != level:
            raise ValueError("slab level mismatch")
        self.h = hydro or HydroConfig()
        self.g = gravity or GravityConfig(expansion_order=1)
        self.group = group
        # gravity arithmetic: "exact" = bit-identical to the reference;
        # "fma" = FMA-contracted far/near terms within 1e-12 (include/sg.h)
        if precision not in ("exact", "fma"):
            raise ValueError(f"precision must be 'exact' or 'fma', got {precision!r}")
        self.precision = precision
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise ValueError(f"UnigridState needs a CUDA device, got {self.device}")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        n, nz = self.slab.n, self.slab.nz
        self.n, self.nz = n, nz
        self.dx = 1.0 / n
        self.halo = gravity_halo(self.g.theta)
        self.rad2, self.eps2 = gravity_params(self.dx, self.g)
        f64 = dict(dtype=torch.float64, device=self.device)
        self.uv = View(n, n, nz, U_PAD)
        self.mv = View(n, n, nz, MASS_PAD)
        self.gv = View(n, n, nz, 0)
        self.U = torch.zeros((5,) + self.uv.padded_shape, **f64)
        self.mass = torch.zeros(self.mv.padded_shape, **f64)
        mz, my, mx = self.mv.padded_shape
        self.clusters = torch.zeros((mz // 2, my // 2, mx // 2, 4), **f64)
        self.grav = torch.zeros((4, nz, n, n), **f64)
        self.leaves_host = self.slab.leaf_coords()
        self.leaves = self.leaves_host.to(self.device)
        self.nleaves = len(self.leaves_host)
        nb = self.nleaves
        # fused reconstruct+flux never materialises Q; the unfused (drop-in
        # kernel pair) path allocates it lazily
        self.fused_hydro = fused_hydro and not legacy_flux
        self.legacy_flux = legacy_flux   # reference kernels/legacy.py flux formulation
        self._Q = None
        self.FX = torch.empty((nb, 5, 8, 8, 9), **f64)
        self.FY = torch.empty((nb, 5, 8, 9, 8), **f64)
        self.FZ = torch.empty((nb, 5, 9, 8, 8), **f64)
        self.smax = torch.empty(nb, **f64)
        self.ws = torch.empty(nb, **f64)
        self.s_pre = torch.zeros(1, **f64)
        self.dt = torch.zeros(1, **f64)
        i32 = dict(dtype=torch.int32, device=self.device)
        self.flux_err = torch.empty(nb, **i32)
        self.upd_status = torch.empty(nb, **i32)
        self.flux_latch = torch.full((nb,), -1, **i32)     # 0xFFFFFFFF
        self.upd_latch = torch.full((nb,), -1, **i32)
        # first failing hydro iteration (include/sg.h, sg_flux `gate`): the
        # reference raises right after it (driver.py:173-174), so errors of
        # later iterations are not latched; err_info keeps that iteration's
        # (smax, dt) per failing leaf for the CFL message
        self.err_gate = torch.full((1,), GATE_OPEN, **i32)
        self.err_info = torch.zeros((nb, 2), **f64)
        self.hydro_iter = 0      # hydro iterations launched since load()
        self.step_index = 0      # timesteps started since load()
        self._iter_step = []     # hydro iteration -> timestep index
        self.timers = None  # optional {kernel: [(start, end) events]} for per-kernel timing
        # P2P beside M2L on a side stream (see gravity_kernels); its launches
        # are not timed then (an event pair would include the wait for the
        # M2L tail)
        self.overlap_p2p = os.environ.get("SG_P2P_OVERLAP", "1") != "0"  # "0": serial (A/B tooling)
        self._side = None
        self._grav_p2p = None
        self._p2p_side = False   # the last gravity iteration ran P2P on the side stream

    # -- host <-> device ---------------------------------------------------

    @_on_device
    def load(self, state: dict, *, global_arrays: bool = True) -> None:
        """Upload rho, sx, sy, sz, E (global (n,n,n) arrays, or this slab's
        (nz,n,n) part when global_arrays is False)."""
        z0, nz, p = self.slab.z0, self.nz, U_PAD
        for v, name in enumerate(HYDRO_FIELDS):
            a = np.asarray(state[name], dtype=np.float64)
            if global_arrays:
                a = a[z0:z0 + nz]
            self.U[v, p:p + nz, p:p + self.n, p:p + self.n].copy_(torch.from_numpy(np.ascontiguousarray(a)))
        self.reset_errors()

    @_on_device
    def fetch(self) -> dict:
        p = U_PAD
        U = self.U[:, p:p + self.nz, p:p + self.n, p:p + self.n].cpu().numpy()
        out = {name: U[v] for v, name in enumerate(HYDRO_FIELDS)}
        g = self.grav.cpu().numpy()
        for i, name in enumerate(("phi", "gx", "gy", "gz")):
            out[name] = g[i]
        return out

    @property
    def Q(self) -> torch.Tensor:
        if self._Q is None:
            self._Q = torch.empty((self.nleaves, 5, 26, 1000), dtype=torch.float64, device=self.device)
        return self._Q

    # -- octree <-> device ------------------------------

    @classmethod
    def from_tree(cls, tree, hydro: HydroConfig | None = None, gravity: GravityConfig | None = None,
                  **kw) -> "UnigridState":
        """Device-resident state of a (reference or local) unigrid Octree: the
        leaves' interiors become the padded global fields."""
        from .octree import global_field
        st = cls(tree.max_level, hydro, gravity, **kw)
        st.load({name: global_field(tree, name) for name in HYDRO_FIELDS})
        return st

    def to_tree(self, tree, names=HYDRO_FIELDS + ("phi", "gx", "gy", "gz")) -> None:
        """Write the device state back into the tree's leaf interiors."""
        from .octree import set_global_field
        if self.slab.world != 1:
            raise ValueError("to_tree needs the whole domain (single slab)")
        out = self.fetch()
        for name in names:
            set_global_field(tree, name, out[name])

    @_on_device
    def source_cubes(self, field: str = "mass", halo: int = 8, leaf_ids=None) -> torch.Tensor:
        """Batched octree.source_cube on the device: (B, 8+2h, 8+2h, 8+2h)
        boxes of `mass` (pad 8) or of a hydro variable (pad 2), after the
        periodic fill.  leaf_ids index self.leaves (default: all)."""
        if field == "mass":
            f, v, ncomp = self.mass, self.mv, 1
        else:
            f, v, ncomp = self.U[HYDRO_FIELDS.index(field)], self.uv, 1
        self._halo(f.view((ncomp,) + v.padded_shape), ncomp, v)
        leaves = self.leaves if leaf_ids is None else self.leaves[torch.as_tensor(leaf_ids, device=self.device)]
        leaves = leaves.contiguous()
        S = 8 + 2 * halo
        out = torch.empty((len(leaves), S, S, S), dtype=torch.float64, device=self.device)
        B.gather_blocks(f, v, leaves, len(leaves), 1, halo, out)
        return out

    @_on_device
    def reset_errors(self) -> None:
        self.flux_latch.fill_(-1)
        self.upd_latch.fill_(-1)
        self.err_gate.fill_(GATE_OPEN)
        self.hydro_iter = 0
        self.step_index = 0
        self._iter_step = []

    # -- per-kernel timing hooks -------------------------------------------

    def _t(self, name: str):
        if self.timers is None:
            return None
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
        self.timers.setdefault(name, []).append(ev)
        return ev[1]

    @staticmethod
    def _done(ev) -> None:
        if ev is not None:
            ev.record()

    # -- ghost / halo ------------------------------------------------------

    def _halo(self, field: torch.Tensor, ncomp: int, view: View) -> None:
        if self.slab.world == 1:
            B.fill_periodic(field, ncomp, view, 7)
        else:
            B.fill_periodic(field, ncomp, view, 3)
            exchange_z_halo(field.view((ncomp,) + view.padded_shape), view.pad, self.slab, self.group)

    # -- the step pieces ---------------------------------------------------

    @_on_device
    def set_mass(self) -> None:
        """driver.py:165-166: mass = rho * dx**3 (Python float pow, as the reference)."""
        B.scale_copy(self.mass, MASS_PAD, self.U, U_PAD, self.n, self.n, self.nz, self.dx ** 3)

    @_on_device
    def gravity_iteration(self) -> None:
        """driver.py:168-169: ghost exchange, then monopole and multipole for
        every leaf; the multipole result overwrites the monopole one in the
        shared phi/g outputs exactly as in the reference."""
        self._halo(self.mass, 1, self.mv)
        self.gravity_kernels()

    @_on_device
    def gravity_kernels(self) -> None:
        """cluster aggregation, P2P and M2L of one gravity iteration.

        In the reference the monopole result is overwritten by the multipole
        one (driver.py:123-139): P2P's output is dead, its inputs are M2L's.
        So P2P runs on a side stream into its own buffer (p2p_result()),
        launched right after M2L: the persistent M2L kernel holds every SM
        (one CTA filling the register file) and P2P's CTAs take the SMs the
        M2L tail leaves idle (4096 subgrids = 27 full rounds + 100 on 148
        SMs).  The main stream waits for P2P before anything that rewrites
        the masses.  Same work, same bits in phi/g."""
        ev = self._t("cluster_aggregate")
        B.cluster_aggregate(self.mass, self.dx, self.clusters)
        self._done(ev)
        self._p2p_side = self.overlap_p2p
        if not self.overlap_p2p:
            ev = self._t("p2p")
            B.p2p(self.mass, self.mv, self.leaves, self.nleaves, self.dx, self.rad2, self.eps2, self.halo,
                  self.grav, self.gv, precision=self.precision)
            self._done(ev)
            self._m2l()
            return
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.device)
            self._ev_in = torch.cuda.Event()
            self._ev_p2p = torch.cuda.Event()
            self._grav_p2p = torch.empty_like(self.grav)
        main = torch.cuda.current_stream(self.device)
        self._ev_in.record(main)
        self._m2l()
        self._side.wait_event(self._ev_in)
        with torch.cuda.stream(self._side):
            B.p2p(self.mass, self.mv, self.leaves, self.nleaves, self.dx, self.rad2, self.eps2, self.halo,
                  self._grav_p2p, self.gv, precision=self.precision)
            self._ev_p2p.record(self._side)
        main.wait_event(self._ev_p2p)

    def _m2l(self) -> None:
        ev = self._t("m2l")
        B.m2l(self.mass, self.mv, self.clusters, 0, self.leaves, self.nleaves, self.dx, self.rad2, self.eps2,
              self.g.expansion_order, self.grav, self.gv, precision=self.precision)
        self._done(ev)

    def p2p_result(self) -> torch.Tensor | None:
        """(phi, gx, gy, gz) of the last gravity iteration's P2P (monopole)
        pass, which phi/g (the multipole result) overwrite in the reference;
        None when that iteration ran serially (its P2P output went to phi/g
        and was overwritten there, as in the reference)."""
        return self._grav_p2p if self._p2p_side else None

    @_on_device
    def wavespeed_dt(self) -> None:
        """driver.py:170-171 on device (+ MAX all-reduce across slabs)."""
        self.wavespeed_local()
        allreduce_max_(self.s_pre, self.slab, self.group)
        B.dt_from_smax(self.s_pre, self.h.cfl, self.dx, self.dt)

    @_on_device
    def wavespeed_local(self) -> None:
        ev = self._t("max_wavespeed")
        B.max_wavespeed(self.U, self.uv, self.leaves, self.nleaves, self.h.gamma, self.h.positivity_floor,
                        self.ws)
        B.max_reduce(self.ws, self.nleaves, self.s_pre)
        self._done(ev)

    @_on_device
    def hydro_iteration(self) -> None:
        """driver.py:173-174 / hydro_job 141-160 for every leaf."""
        self._halo(self.U, 5, self.uv)
        self.hydro_kernels()

    @_on_device
    def hydro_kernels(self) -> None:
        it = self.hydro_iter
        if it >= GATE_OPEN:
            raise OverflowError("hydro iteration counter exhausted; call load() or reset_errors()")
        self.hydro_iter += 1
        self._iter_step.append(self.step_index)
        gate = dict(gate=self.err_gate, it=it)
        if self.fused_hydro:
            ev = self._t("hydro_fused")
            B.hydro_fused(self.U, self.uv, self.leaves, self.nleaves, self.h.positivity_floor, self.h.gamma,
                          self.FX, self.FY, self.FZ, self.smax, self.flux_err, self.flux_latch, **gate)
            self._done(ev)
        else:
            ev = self._t("reconstruct")
            B.reconstruct(self.U, self.uv, self.leaves, self.nleaves, self.h.positivity_floor, self.Q)
            self._done(ev)
            ev = self._t("flux")
            fl = B.flux_legacy if self.legacy_flux else B.flux
            fl(self.Q, self.nleaves, self.h.gamma, self.FX, self.FY, self.FZ, self.smax, self.flux_err,
               self.flux_latch, **gate)
            self._done(ev)
        ev = self._t("hydro_update")
        B.hydro_update(self.U, self.uv, self.leaves, self.nleaves, self.FX, self.FY, self.FZ, self.smax,
                       self.dt, 0.0, self.dx, self.h.cfl, self.upd_status, self.upd_latch, err_info=self.err_info,
                       **gate)
        self._done(ev)

    @_on_device
    def step(self, gravity_per_step: int = 6, hydro_per_step: int = 3) -> None:
        """One reference timestep (driver.py:163-174).  Errors are latched on
        the device (first failing hydro iteration only); check_errors()
        raises them, with that iteration's step number, at any later time."""
        if gravity_per_step:
            self.set_mass()
            for _ in range(gravity_per_step):
                self.gravity_iteration()
        self.wavespeed_dt()
        for _ in range(hydro_per_step):
            self.hydro_iteration()
        self.step_index += 1

    # -- errors --------------------------------------------------------------

    @_on_device
    def check_errors(self, step: int | None = None) -> None:
        """Raise the reference's KernelError for the first failing hydro
        iteration's first failing leaf in Morton (leaf_iter) order, prefixed
        "step N: " like driver._join (driver.py:83-88).  `step` overrides the
        recorded step number."""
        gate = int(self.err_gate.item())
        if self.slab.world > 1:  # every rank raises the global first error
            gate = allreduce_min_int(gate, self.slab, self.group)
            if gate == GATE_OPEN:
                return
            first = self._first_error(step, gate)
            c = first_error_across_ranks(None if first is None else (first[0], str(first[1])), self.slab,
                                         self.group)
            first = None if c is None else (c[0], KernelError(c[1]))
        else:
            first = self._first_error(step, gate)
        if first is not None:
            raise first[1]

    def failing_iteration(self) -> int | None:
        """Index (since load()) of the first failing hydro iteration, or None."""
        g = int(self.err_gate.item())
        return None if g == GATE_OPEN else g

    @_on_device
    def _first_error(self, step: int | None = None, gate: int | None = None):
        """(Morton key, KernelError) of this slab's first failing leaf in the
        first failing hydro iteration `gate` (default: this slab's), or None."""
        own = int(self.err_gate.item())
        gate = own if gate is None else gate
        if gate == GATE_OPEN or own != gate:  # no error here in that iteration
            return None
        fl = self.flux_latch.cpu().numpy().view(np.uint32)
        up = self.upd_latch.cpu().numpy().view(np.uint32)
        bad = np.nonzero((fl != B.U32_OK) | (up != B.U32_OK))[0]
        if not len(bad):
            return None
        coords = self.slab.global_leaf_coords().numpy()
        key = lambda i: morton_key(*coords[i], self.level)  # noqa: E731
        b = min(bad, key=key)
        coord = tuple(int(c) for c in coords[b])
        if step is None and gate < len(self._iter_step):
            step = self._iter_step[gate]
        prefix = f"step {step}: " if step is not None else ""
        if fl[b] != B.U32_OK:
            code, cell = decode_flux_error(int(fl[b]))
            what = "density" if code == 1 else "pressure"
            return key(b), KernelError(f"{prefix}non-positive {what} at a quadrature point of cell "
                                       f"(x={cell % 10 + 1}, y={(cell // 10) % 10 + 1}, z={cell // 100 + 1}) "
                                       f"[extended indices] of leaf {coord}")
        kind, detail = int(up[b]) >> 16, int(up[b]) & 0xFFFF
        smax, dt = (float(v) for v in self.err_info[b].tolist())  # that iteration's values
        if kind == 0:
            return key(b), KernelError(f"{prefix}dt must be positive, got {dt}")
        if kind == 1:  # message of reference kernels/__init__.py:170-174
            return key(b), KernelError(f"{prefix}CFL violation: dt={dt:g} exceeds cfl*dx/s_max="
                                       f"{self.h.cfl * self.dx / smax:g} (s_max={smax:g})")
        name = "rho" if kind == 2 else "E"
        return key(b), KernelError(f"{prefix}non-positive (or NaN) {name} after update at interior cell "
                                   f"(x={detail % 8}, y={(detail // 8) % 8}, z={detail // 64}) of leaf {coord}")


class HostPipeline:
    """Host-buffer stepping with copy/compute overlap: each ``submit`` takes a
    pinned host state (5, nz, n, n), runs one timestep on it and returns the
    new state plus gravity (9, nz, n, n) into a pinned host buffer.  Uploads
    and readbacks run on copy streams through double-buffered device
    staging, so submission k's transfers overlap the compute of k-1 / k+1
    (independent inputs, e.g. ensembles or a stream of snapshots).  Results
    are those of ``UnigridState.load`` + ``step`` + ``fetch``."""

    def __init__(self, state: UnigridState):
        self.st = state
        dev = state.device
        shp = (5, state.nz, state.n, state.n)
        f64 = dict(dtype=torch.float64, device=dev)
        self.u_in = [torch.empty(shp, **f64) for _ in range(2)]
        self.out = [torch.empty((9,) + shp[1:], **f64) for _ in range(2)]
        # separate upload and download streams: on one FIFO stream upload k+1
        # would queue behind readback k, which waits for step k to finish
        self.up = torch.cuda.Stream(device=dev)
        self.down = torch.cuda.Stream(device=dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_in_free = [torch.cuda.Event() for _ in range(2)]
        self.ev_result = [torch.cuda.Event() for _ in range(2)]
        self.ev_out_free = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_in_free + self.ev_out_free:
            e.record()
        self.k = 0

    def submit(self, host_in: torch.Tensor, host_out: torch.Tensor, **step_kw) -> torch.cuda.Event:
        st, i = self.st, self.k % 2
        p, nz, n = U_PAD, st.nz, st.n
        comp = torch.cuda.current_stream(st.device)
        with torch.cuda.stream(self.up):
            self.up.wait_event(self.ev_in_free[i])
            self.u_in[i].copy_(host_in, non_blocking=True)
            self.ev_h2d[i].record(self.up)
        comp.wait_event(self.ev_h2d[i])
        st.U[:, p:p + nz, p:p + n, p:p + n].copy_(self.u_in[i])
        self.ev_in_free[i].record(comp)
        st.step(**step_kw)
        comp.wait_event(self.ev_out_free[i])
        self.out[i][:5].copy_(st.U[:, p:p + nz, p:p + n, p:p + n])
        self.out[i][5:].copy_(st.grav)
        self.ev_result[i].record(comp)
        with torch.cuda.stream(self.down):
            self.down.wait_event(self.ev_result[i])
            host_out.copy_(self.out[i], non_blocking=True)
            self.ev_out_free[i].record(self.down)
        self.k += 1
        return self.ev_out_free[i]

    def synchronize(self) -> None:
        self.up.synchronize()
        self.down.synchronize()
        torch.cuda.current_stream(self.st.device).synchronize()


class LocalSlabs:
    """The z-slab decomposition with all P slabs in one process on one
    device: same kernels, same halo planes as the NCCL path, exchanged by
    device copies.  Used to check that results are bitwise P-invariant."""

    def __init__(self, level: int, world: int, hydro: HydroConfig | None = None,
                 gravity: GravityConfig | None = None):
        self.states = [UnigridState(level, hydro, gravity, slab=Slab(level, r, world)) for r in range(world)]
        self.world = world

    def load(self, state: dict) -> None:
        for s in self.states:
            s.load(state)

    def _halo_all(self, name: str, ncomp: int, view: View) -> None:
        fields = []
        for s in self.states:
            f = getattr(s, name)
            B.fill_periodic(f, ncomp, view, 3)
            fields.append(f.view((ncomp,) + view.padded_shape))
        exchange_z_halo_local(fields, view.pad, self.states[0].nz)

    def step(self, gravity_per_step: int = 6, hydro_per_step: int = 3) -> None:
        st = self.states
        if gravity_per_step:
            for s in st:
                s.set_mass()
            for _ in range(gravity_per_step):
                self._halo_all("mass", 1, st[0].mv)
                for s in st:
                    s.gravity_kernels()
        for s in st:
            s.wavespeed_local()
        s_pre = torch.stack([s.s_pre for s in st]).max(dim=0).values
        for s in st:
            s.s_pre.copy_(s_pre)
            B.dt_from_smax(s.s_pre, s.h.cfl, s.dx, s.dt)
        for _ in range(hydro_per_step):
            self._halo_all("U", 5, st[0].uv)
            for s in st:
                s.hydro_kernels()
        for s in st:
            s.step_index += 1

    def check_errors(self, step: int | None = None) -> None:
        """The first failing hydro iteration over all slabs, and in it the
        first failing leaf in global Morton order (the reference's leaf_iter
        order interleaves z)."""
        gate = min(int(s.err_gate.item()) for s in self.states)
        found = [e for e in (s._first_error(step, gate) for s in self.states) if e is not None]
        if found:
            raise min(found, key=lambda e: e[0])[1]

    def fetch(self) -> dict:
        parts = [s.fetch() for s in self.states]
        return {k: np.concatenate([p[k] for p in parts], axis=0) for k in parts[0]}


def run_steps(state: dict, level: int, steps: int, *, hydro: HydroConfig | None = None,
              gravity: GravityConfig | None = None, gravity_per_step: int = 6, slab: Slab | None = None,
              group=None, check_every_step: bool = True, precision: str = "exact") -> tuple[dict, list]:
    """Public end-to-end entry: host arrays in, ``steps`` reference timesteps on
    the device, host arrays out (plus the per-step dt values)."""
    st = UnigridState(level, hydro, gravity, slab=slab, group=group, precision=precision)
    st.load(state)
    dts = []
    for s in range(steps):
        st.step(gravity_per_step)
        dts.append(st.dt.item() if check_every_step else None)
        if check_every_step:
            st.check_errors(s)
    st.check_errors()
    return st.fetch(), dts

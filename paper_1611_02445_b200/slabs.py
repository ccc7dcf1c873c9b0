"""Multi-GPU z-slab decomposition over tile layers.

One process per GPU.  The global geometry is cut along z into slabs of whole
4-node tile layers, balanced by non-solid node count.  Every rank builds the
local geometry ``[ghost layer | owned layers | ghost layer]`` (the ghost layers
are copies of the neighbours' boundary layers; with a periodic z axis the
first and last ranks are neighbours) and runs the ordinary device tiler and
step on it.  Because the tile list is z-outermost (tiling.py:70-75), the owned
tiles are one contiguous index range and each layer is a sub-range, so the
step kernel is simply launched on tile ranges.

Per step (copy p -> 1-p):
  1. step the owned bottom and top tile layers          (boundary)
  2. pack their outgoing z planes (80 values per tile: 5 directions x 16
     nodes; csrc/fields.cu tlbm_halo)
  3. exchange with the z neighbours (NCCL send/recv on NCCL's stream, or
     device copies between virtual ranks on one GPU)
  4. step the interior layers -- concurrently with 3
  5. unpack into the ghost layers of copy 1-p, flip parity
Ghost node *tags* never change, so they are part of the local geometry and
the per-node link masks of owned nodes are exact; only f values move.

The exchange moves 640 B (fp64) per boundary tile per direction of travel;
results are bit-identical to the single-domain run (tests).
"""

from dataclasses import dataclass

import ctypes

import numpy as np
import torch

from . import _native as nat
from .geometry import Geometry
from .solver import SimulationConfig, Solver, use_nodes
from .tiling import DeviceTiling

TILE = 4


@dataclass
class SlabRange:
    rank: int
    z0: int                 # first owned node layer (global)
    z1: int                 # one past the last owned node layer (global)
    lower: int              # rank owning the layer below (-1: none)
    upper: int              # rank owning the layer above (-1: none)


class SlabPlan:
    """Partition of the global z extent into per-rank tile-layer ranges."""

    def __init__(self, geometry, world):
        nx, ny, nz = geometry.shape
        self.world = int(world)
        self.dims = (nx, ny, nz)
        self.periodic_z = bool(geometry.periodic[2])
        ntz = -(-nz // TILE)
        if self.world < 1 or self.world > ntz:
            raise ValueError(f"cannot cut {ntz} tile layers into {world} slabs")
        if self.periodic_z and self.world > 1 and nz % TILE:
            raise ValueError("periodic z needs a multiple of 4 layers")
        if self.world == 1:
            self.layer_weight = None
            self.ranges = [SlabRange(0, 0, nz, -1, -1)]
            return
        # non-solid node count per tile layer -> balanced contiguous cuts
        ns = np.count_nonzero(geometry.types, axis=(0, 1))
        pad = np.zeros(ntz * TILE, dtype=np.int64)
        pad[:nz] = ns
        per_layer = pad.reshape(ntz, TILE).sum(1)
        self.layer_weight = per_layer
        cum = np.concatenate([[0], np.cumsum(per_layer)])
        total = cum[-1]
        cuts = [0]
        for r in range(1, self.world):
            target = total * r / self.world
            c = int(np.searchsorted(cum, target))
            if c > 0 and abs(cum[c - 1] - target) <= abs(cum[min(c, ntz)] - target):
                c -= 1                      # nearest prefix boundary to the target
            c = min(max(c, cuts[-1] + 1), ntz - (self.world - r))
            cuts.append(c)
        cuts.append(ntz)
        self.ranges = []
        for r in range(self.world):
            lower = r - 1 if r > 0 else (self.world - 1 if self.periodic_z and self.world > 1
                                         else -1)
            upper = r + 1 if r < self.world - 1 else (0 if self.periodic_z and self.world > 1
                                                     else -1)
            self.ranges.append(SlabRange(r, cuts[r] * TILE, min(cuts[r + 1] * TILE, nz),
                                         lower, upper))

    def local_types(self, types, rank):
        """[ghost below | owned | ghost above] tags of one rank."""
        r = self.ranges[rank]
        nz = self.dims[2]
        parts = []
        if r.lower >= 0:
            lo = r.z0 - TILE
            parts.append(types[:, :, lo:r.z0] if lo >= 0 else types[:, :, nz - TILE:nz])
        parts.append(types[:, :, r.z0:r.z1])
        if r.upper >= 0:
            # the layer above; it wraps to z = 0..3 only across the periodic
            # seam (r.z1 == nz).  A last layer of fewer than 4 nodes (nz % 4
            # != 0, never periodic) is a partial ghost padded with SOLID.
            parts.append(types[:, :, r.z1:min(r.z1 + TILE, nz)] if r.z1 < nz
                         else types[:, :, 0:TILE])
        return np.ascontiguousarray(np.concatenate(parts, axis=2))

    def local_geometry(self, geometry, rank):
        if self.world == 1:
            return geometry
        per = tuple(geometry.periodic)
        if self.world > 1:
            per = (per[0], per[1], False)
        return Geometry(self.local_types(geometry.types, rank), geometry.inlet_velocity,
                        geometry.outlet_density, periodic=per)


def layer_tile_ranges(tile_map):
    """[begin, end) tile-index range of every local tile layer (tz)."""
    occ = (tile_map >= 0).sum(axis=(0, 1)) if isinstance(tile_map, np.ndarray) else \
        (tile_map >= 0).sum(dim=(0, 1)).cpu().numpy()
    ends = np.cumsum(occ)
    begins = ends - occ
    return [(int(b), int(e)) for b, e in zip(begins, ends)]


def resolve_auto_storage_global(config, geometry):
    """storage="auto" decided on the whole geometry's tile utilisation, so
    that every slab rank picks the same storage."""
    from .solver import resolve_auto_storage
    t = np.asarray(geometry.types) != 0
    mesh = tuple(-(-n // TILE) for n in t.shape)
    occ = np.zeros(tuple(m * TILE for m in mesh), dtype=bool)
    occ[:t.shape[0], :t.shape[1], :t.shape[2]] = t
    t_n = int(occ.reshape(mesh[0], TILE, mesh[1], TILE, mesh[2], TILE).any(axis=(1, 3, 5)).sum())
    return resolve_auto_storage(config, int(t.sum()), t_n)


class SlabSolver:
    """One rank's slab: a local Solver plus the halo bookkeeping."""

    def __init__(self, geometry, plan, rank, config=None, device=None, traversal="auto",
                 initial=(1.0, (0.0, 0.0, 0.0))):
        """``traversal``: "tile" (tile-parallel step), "nodes" (node-parallel
        step over the nodes of each launched tile range; compact storage) or
        "auto" (solver.use_nodes)."""
        self.plan, self.rank = plan, rank
        self.range = plan.ranges[rank]
        self.local_geometry = plan.local_geometry(geometry, rank)
        if config is not None and config.storage == "auto":
            # every rank must use the same storage (the fused halo writes into
            # the neighbour's store): decide on the whole geometry
            config = resolve_auto_storage_global(config, geometry)
        # slab launches name tile ranges (boundary layers, interior), so the
        # solver keeps the tile-list order (or runs node-parallel over the
        # nodes of those ranges)
        config = config or SimulationConfig()
        tiling = DeviceTiling(self.local_geometry, device)
        if traversal not in ("tile", "nodes"):
            traversal = ("nodes" if use_nodes(config, tiling.n_fn, tiling.t_n, "auto")
                         else "tile")
        self.solver = Solver(self.local_geometry, config, device, tiling=tiling,
                             traversal=traversal, initial=initial)
        s = self.solver
        layers = layer_tile_ranges(s.tiling.tile_map)
        has_lo, has_hi = self.range.lower >= 0, self.range.upper >= 0
        own = layers[(1 if has_lo else 0):(len(layers) - 1 if has_hi else len(layers))]
        self.ghost_lo = layers[0] if has_lo else None
        self.ghost_hi = layers[-1] if has_hi else None
        self.own = (own[0][0], own[-1][1])
        self.bottom, self.top = own[0], own[-1]
        self.interior = (self.bottom[1], self.top[0]) if len(own) > 2 else (self.top[0],
                                                                            self.top[0])
        self.n_fn_owned = int(s.tiling.counts[self.own[0]:self.own[1]].sum().item())
        self._side = None
        self._n_over = 0
        dt = s.store.tdtype
        dev = s.device
        nb = lambda r: torch.empty(max(r[1] - r[0], 0) * 80, dtype=dt, device=dev)  # noqa
        self.send_up = nb(self.top) if has_hi else None
        self.send_down = nb(self.bottom) if has_lo else None
        self.recv_lo = nb(self.ghost_lo) if has_lo else None
        self.recv_hi = nb(self.ghost_hi) if has_hi else None
        if has_lo and self.recv_lo.numel() != (self.ghost_lo[1] - self.ghost_lo[0]) * 80:
            raise AssertionError("ghost layer size mismatch")

    # -- the pieces of one step ---------------------------------------------
    def _launch(self, rng):
        if rng[1] > rng[0]:
            s = self.solver
            a = s._args
            a.tile_begin, a.tile_end = rng
            if s.nodes is not None:
                a.node_begin, a.node_end = s.store.node_range(*rng)
            a.f_src = s._copies[s.parity]
            a.f_dst = s._copies[1 - s.parity]
            a.flags = s.status.data_ptr() + 4 * (s.iteration % len(s.status))
            nat.check(nat.load().tlbm_step(nat.ctypes.byref(a), nat.stream_ptr(s.device)))

    def step_boundary(self):
        self._launch(self.bottom)
        if self.top != self.bottom:
            self._launch(self.top)

    def step_interior(self):
        self._launch(self.interior)

    # -- interior / boundary overlap on two streams --------------------------
    def step_overlapped(self, before=None, after=None, wait_events=()):
        """One step with the interior tiles on the current stream and the
        boundary layers on a high-priority side stream, so they run
        concurrently (the boundary launches fill the interior's tail instead
        of following it).  ``before`` / ``after`` run on the side stream
        around the boundary launches (peer wait + arm / disarm + signal);
        ``wait_events`` are extra events the side stream waits on first.

        Ordering, step t: the interior waits for boundary t-1 (it reads the
        boundary tiles t-1 wrote, and writes the copy boundary t-1 read); the
        boundary waits for everything the current stream had before interior
        t, i.e. interior t-1 (same reasons).  Interior t and boundary t read
        the same copy and write disjoint tiles of the other."""
        dev = self.solver.device
        if self._side is None:
            self._side = torch.cuda.Stream(device=dev, priority=-1)
            self._ev_pre = [torch.cuda.Event(), torch.cuda.Event()]
            self._ev_bnd = [torch.cuda.Event(), torch.cuda.Event()]
        main = torch.cuda.current_stream(dev)
        t = self._n_over
        if t > 0:
            main.wait_event(self._ev_bnd[(t - 1) % 2])
        self._ev_pre[t % 2].record(main)
        self.step_interior()
        with torch.cuda.stream(self._side):
            self._side.wait_event(self._ev_pre[t % 2])
            for ev in wait_events:
                self._side.wait_event(ev)
            if before is not None:
                before()
            self.step_boundary()
            if after is not None:
                after()
            self._ev_bnd[t % 2].record(self._side)
        self._n_over += 1

    def last_boundary_event(self):
        return self._ev_bnd[(self._n_over - 1) % 2] if self._n_over > 0 else None

    def join(self):
        """Make the current stream wait for the side stream's last boundary
        launch (before any host read or non-overlapped launch)."""
        if self._n_over > 0:
            torch.cuda.current_stream(self.solver.device).wait_event(
                self._ev_bnd[(self._n_over - 1) % 2])
            self._n_over = 0

    def _halo(self, rng, up, pack, buf, copy):
        s = self.solver
        st = s.store
        if s.config.storage == "compact":
            nat.call("tlbm_halo_compact", nat.ptr(st.copy_tensor(copy)), s.code, rng[0], rng[1],
                     int(up), int(pack), nat.ptr(buf), nat.ptr(st.base), nat.ptr(st.nf),
                     nat.ptr(st.rank), nat.stream_ptr(s.device))
            return
        nat.call("tlbm_halo", nat.ptr(st.copy_tensor(copy)), s.code, s.table,
                 rng[0], rng[1], int(up), int(pack), nat.ptr(buf), nat.stream_ptr(s.device))

    @property
    def compact(self):
        return self.solver.config.storage == "compact"

    def ghost_cbase(self, which):
        """Block offsets of the ghost layer ``which`` ("lo" | "hi") of a
        compact store (where a neighbour's fused halo writes)."""
        g = self.ghost_lo if which == "lo" else self.ghost_hi
        return self.solver.store.base[g[0]:g[1]]

    def pack(self, current=False):
        """Pack the outgoing planes of the copy just written (or, with
        ``current``, of the current copy -- the initial ghost fill)."""
        c = self.solver.parity if current else 1 - self.solver.parity
        if self.send_up is not None:
            self._halo(self.top, True, True, self.send_up, c)
        if self.send_down is not None:
            self._halo(self.bottom, False, True, self.send_down, c)

    def unpack(self, current=False):
        c = self.solver.parity if current else 1 - self.solver.parity
        if self.recv_lo is not None:
            self._halo(self.ghost_lo, True, False, self.recv_lo, c)
        if self.recv_hi is not None:
            self._halo(self.ghost_hi, False, False, self.recv_hi, c)

    def finish(self):
        s = self.solver
        s.parity ^= 1
        s.iteration += 1
        if s.iteration - s._checked >= len(s.status) - 1:
            self.join()
            s.check()

    def fields_owned(self):
        """Canonical (19, t_own, 64) of the owned tiles (current copy)."""
        f = self.solver.fields_canonical(device=True)
        return f[:, self.own[0]:self.own[1]]


class NcclHalo:
    """Neighbour exchange over torch.distributed (NCCL on GPUs).

    Fixed post order on every rank -- sends [up, down], receives [from below,
    from above] -- so that, with two ranks and periodic z, both messages to
    the same peer match in order."""

    def __init__(self, slab):
        import torch.distributed as dist
        self.dist, self.slab = dist, slab

    def start(self):
        d, sl, r = self.dist, self.slab, self.slab.range
        ops = []
        if sl.send_up is not None:
            ops.append(d.P2POp(d.isend, sl.send_up, r.upper))
        if sl.send_down is not None:
            ops.append(d.P2POp(d.isend, sl.send_down, r.lower))
        if sl.recv_lo is not None:
            ops.append(d.P2POp(d.irecv, sl.recv_lo, r.lower))
        if sl.recv_hi is not None:
            ops.append(d.P2POp(d.irecv, sl.recv_hi, r.upper))
        return d.batch_isend_irecv(ops) if ops else []

    @staticmethod
    def wait(reqs):
        for q in reqs:
            q.wait()


def _export(t):
    h = (ctypes.c_char * 64)()
    off = ctypes.c_uint64(0)
    nat.call("tlbm_ipc_export", nat.ptr(t), h, ctypes.byref(off))
    return bytes(h), int(off.value)


def _import(handle, offset):
    p = ctypes.c_void_p(0)
    buf = (ctypes.c_char * 64).from_buffer_copy(handle)
    nat.call("tlbm_ipc_import", buf, ctypes.c_uint64(offset), ctypes.byref(p))
    return int(p.value), int(p.value) - offset          # (pointer, mapping base)


class IpcHalo:
    """Fused halo over peer memory (CUDA IPC; NVLink between GPUs).

    The boundary-layer step kernel stores its outgoing z planes directly
    into the neighbours' ghost tiles (tlbm_step_args.halo_*): no pack kernel,
    no staging buffer, no copy engine, no NCCL on the step path.  Ordering is
    a stream-ordered step counter per neighbour pair.  Step t runs the
    interior tiles first (own tiles only, no neighbour needed); then the rank
    waits (tlbm_peer_wait) until both neighbours published t, i.e. finished
    the boundary layers of step t-1 -- so their ghost planes of the copy it
    reads are written, and they no longer read the copy whose ghosts it is
    about to write -- runs its boundary layers with the fused peer stores,
    and publishes t+1 into their inboxes (tlbm_peer_signal, system-scope
    fence first).  A wait that exceeds ``timeout_s`` sets an error word and
    returns (checked by ``check``) instead of hanging the GPU.
    """

    def __init__(self, slab, timeout_s=30.0):
        import torch.distributed as dist
        self.dist, self.slab = dist, slab
        s = slab.solver
        r = slab.range
        self.esize = s.store.flat.element_size()
        self.inbox = torch.zeros(2, dtype=torch.int64, device=s.device)  # [from lower, upper]
        self.error = torch.zeros(1, dtype=torch.int32, device=s.device)
        self.timeout_ns = int(timeout_s * 1e9)
        info = {"t_n": s.t_n, "ghost_lo": slab.ghost_lo, "ghost_hi": slab.ghost_hi,
                "top": slab.top, "bottom": slab.bottom, "esize": self.esize,
                "copy_bytes": s.store.copy_tensor(0).numel() * self.esize,
                "compact": slab.compact,
                "ghost_lo_cbase": (slab.ghost_cbase("lo").cpu().tolist()
                                   if slab.compact and slab.ghost_lo else None),
                "ghost_hi_cbase": (slab.ghost_cbase("hi").cpu().tolist()
                                   if slab.compact and slab.ghost_hi else None),
                "store": _export(s.store.flat), "inbox": _export(self.inbox)}
        torch.cuda.synchronize()
        infos = [None] * slab.plan.world
        dist.all_gather_object(infos, info)
        self.bases = []
        mapped = {}
        error = None
        try:
            for nb in sorted({r.lower, r.upper} - {-1}):
                store, b1 = _import(*infos[nb]["store"])
                self.bases.append(b1)
                inbox, b2 = _import(*infos[nb]["inbox"])
                self.bases.append(b2)
                mapped[nb] = (store, inbox)
        except RuntimeError as exc:           # e.g. no P2P path between the GPUs
            error = exc
        # every rank must take the same path (fused halo or fallback), or the
        # collectives that follow would pair up wrongly and hang
        oks = [None] * slab.plan.world
        dist.all_gather_object(oks, error is None)
        if not all(oks):
            for b in self.bases:
                nat.call("tlbm_ipc_close", nat.c_vp(b))
            self.bases = []
            raise RuntimeError(f"peer mapping failed on some rank ({error})")
        tv = 19 * 64 * self.esize
        if any(i["compact"] != slab.compact for i in infos):
            raise AssertionError("slab ranks disagree on the storage")
        dev = s.device
        cb = lambda v: torch.tensor(v, dtype=torch.int64, device=dev)  # noqa: E731
        self.up = self.up_cbase = None
        if r.upper >= 0:
            u = infos[r.upper]
            if u["ghost_lo"][1] - u["ghost_lo"][0] != slab.top[1] - slab.top[0]:
                raise AssertionError("top layer and upper ghost layer differ")
            # (ghost tiles' base, bytes per copy, inbox slot) -- a compact
            # store's ghost tiles are found through their block offsets
            ghost = mapped[r.upper][0] + (0 if slab.compact else u["ghost_lo"][0] * tv)
            self.up = (ghost, u["copy_bytes"], mapped[r.upper][1] + 0)  # upper's "from lower"
            if slab.compact:
                self.up_cbase = cb(u["ghost_lo_cbase"])
        self.down = self.down_cbase = None
        if r.lower >= 0:
            lo = infos[r.lower]
            if lo["ghost_hi"][1] - lo["ghost_hi"][0] != slab.bottom[1] - slab.bottom[0]:
                raise AssertionError("bottom layer and lower ghost layer differ")
            ghost = mapped[r.lower][0] + (0 if slab.compact else lo["ghost_hi"][0] * tv)
            self.down = (ghost, lo["copy_bytes"], mapped[r.lower][1] + 8)  # lower's "from upper"
            if slab.compact:
                self.down_cbase = cb(lo["ghost_hi_cbase"])
        base = self.inbox.data_ptr()
        if r.lower >= 0 and r.upper >= 0:
            self.wait_ptr, self.wait_n = base, 2
        elif r.lower >= 0:
            self.wait_ptr, self.wait_n = base, 1
        elif r.upper >= 0:
            self.wait_ptr, self.wait_n = base + 8, 1
        else:
            self.wait_ptr, self.wait_n = base, 0
        dist.barrier()

    def wait(self, value):
        s = self.slab.solver
        nat.call("tlbm_peer_wait", nat.c_vp(self.wait_ptr), self.wait_n, ctypes.c_uint64(value),
                 ctypes.c_uint64(self.timeout_ns), nat.ptr(self.error), nat.stream_ptr(s.device))

    def arm(self):
        """Point the step args' halo fields at the neighbours' ghost tiles of
        the copy this step writes (parity is the same on every rank)."""
        sl, a = self.slab, self.slab.solver._args
        dst_copy = 1 - sl.solver.parity
        if self.up is not None:
            ghost, copy_bytes, _ = self.up
            a.halo_up = ghost + dst_copy * copy_bytes
            a.halo_up_begin, a.halo_up_end = sl.top
            a.halo_up_cbase = self.up_cbase.data_ptr() if self.up_cbase is not None else None
        if self.down is not None:
            ghost, copy_bytes, _ = self.down
            a.halo_down = ghost + dst_copy * copy_bytes
            a.halo_down_begin, a.halo_down_end = sl.bottom
            a.halo_down_cbase = (self.down_cbase.data_ptr() if self.down_cbase is not None
                                 else None)

    def disarm(self):
        a = self.slab.solver._args
        a.halo_up = a.halo_down = None

    def signal(self, value):
        s = self.slab.solver
        pa = self.up[2] if self.up is not None else None
        pb = self.down[2] if self.down is not None else None
        nat.call("tlbm_peer_signal", nat.c_vp(pa), nat.c_vp(pb), ctypes.c_uint64(value),
                 nat.stream_ptr(s.device))

    def check(self):
        if int(self.error.item()):
            raise RuntimeError("slab neighbour did not reach the step within the timeout")

    def close(self):
        torch.cuda.synchronize()
        self.dist.barrier()
        for b in self.bases:
            nat.call("tlbm_ipc_close", nat.c_vp(b))
        self.bases = []


class HostStagedHalo(NcclHalo):
    """The same exchange through host memory over a CPU process group (gloo):
    lets several ranks share one GPU in tests of the multi-process path."""

    def __init__(self, slab):
        super().__init__(slab)
        sl = slab
        self.h_recv_lo = torch.empty(sl.recv_lo.shape, dtype=sl.recv_lo.dtype) \
            if sl.recv_lo is not None else None
        self.h_recv_hi = torch.empty(sl.recv_hi.shape, dtype=sl.recv_hi.dtype) \
            if sl.recv_hi is not None else None

    def start(self):
        d, sl, r = self.dist, self.slab, self.slab.range
        ops = []
        if sl.send_up is not None:
            ops.append(d.P2POp(d.isend, sl.send_up.cpu(), r.upper))
        if sl.send_down is not None:
            ops.append(d.P2POp(d.isend, sl.send_down.cpu(), r.lower))
        if sl.recv_lo is not None:
            ops.append(d.P2POp(d.irecv, self.h_recv_lo, r.lower))
        if sl.recv_hi is not None:
            ops.append(d.P2POp(d.irecv, self.h_recv_hi, r.upper))
        return (d.batch_isend_irecv(ops) if ops else [], self)

    @staticmethod
    def wait(handle):
        reqs, self = handle
        for q in reqs:
            q.wait()
        if self.h_recv_lo is not None:
            self.slab.recv_lo.copy_(self.h_recv_lo)
        if self.h_recv_hi is not None:
            self.slab.recv_hi.copy_(self.h_recv_hi)


class DistributedSlabRunner:
    """Steps one rank of an N-GPU slab run; NCCL exchange overlapped with the
    interior-tile launch.  ``transport="gloo"`` stages the halo through host
    memory instead (tests with several ranks on one GPU)."""

    def __init__(self, geometry, world, rank, config=None, device=None, transport="nccl",
                 traversal="auto", initial=(1.0, (0.0, 0.0, 0.0))):
        self.plan = SlabPlan(geometry, world)
        self.slab = SlabSolver(geometry, self.plan, rank, config, device, traversal, initial)
        self.transport = transport
        self.ipc = None
        self.halo = None
        if world > 1:
            import torch.distributed as dist
            staged = transport == "gloo" or (transport == "ipc" and
                                              dist.get_backend() == "gloo")
            self.halo = (HostStagedHalo if staged else NcclHalo)(self.slab)
            if transport == "ipc":
                self.ipc = IpcHalo(self.slab)
        self.n_fn_owned = self.slab.n_fn_owned

    def launches_per_step(self):
        """Kernels of this library launched per step (step ranges + halo)."""
        sl = self.slab
        if self.halo is None:
            return 1
        if self.ipc is not None:
            n = 1 if sl.top == sl.bottom else 2
            return n + int(sl.interior[1] > sl.interior[0]) + 2     # + wait + signal
        n = 1 if sl.top == sl.bottom else 2
        n += int(sl.interior[1] > sl.interior[0])
        n += sum(b is not None for b in (sl.send_up, sl.send_down, sl.recv_lo, sl.recv_hi))
        return n

    def exchange_current(self):
        """Fill the ghost planes of the current copy from the neighbours (after
        initialising each rank's fields independently)."""
        if self.halo is None:
            return
        self.slab.pack(current=True)
        self.halo.wait(self.halo.start())
        self.slab.unpack(current=True)

    def step(self, n=1, check=True):
        """Advance n iterations.  ``check`` (default, like Solver.step): read
        the status ring and the peer-wait error word at the end, raising
        DivergenceError / RuntimeError (a neighbour that missed the step)."""
        sl = self.slab
        for _ in range(int(n)):
            if self.halo is None:
                sl._launch(sl.own)
                sl.finish()
                continue
            if self.ipc is not None:
                # interior tiles on the main stream (own tiles only, no
                # neighbour needed); on the high-priority side stream,
                # concurrently: the neighbour wait, the boundary layers with
                # the fused peer stores, and the signal right after them
                it = sl.solver.iteration
                ipc = self.ipc
                sl.step_overlapped(before=lambda: (ipc.wait(it), ipc.arm()),
                                   after=lambda: (ipc.disarm(), ipc.signal(it + 1)))
                sl.finish()
                continue
            sl.step_boundary()
            sl.pack()
            reqs = self.halo.start()
            sl.step_interior()
            self.halo.wait(reqs)
            sl.unpack()
            sl.finish()
        sl.join()
        if check:
            self.check()

    def check(self):
        """Raise on divergence (status ring) or a peer-wait timeout."""
        if self.ipc is not None:
            self.ipc.check()
        self.slab.solver.check()

    def barrier(self):
        if self.halo is not None:
            self.halo.dist.barrier()


class VirtualSlabs:
    """All slabs of a decomposition on ONE device -- exercises the partition,
    halo and ghost logic of the multi-GPU path on a single GPU.

    ``fused=False``: halos move by pack -> device copy -> unpack (the NCCL
    path's data flow).  ``fused=True``: the boundary-layer launches store
    their outgoing planes straight into the neighbour slab's ghost tiles,
    the fused-halo kernels of the IPC path with device pointers in place of
    peer mappings; slabs run one after another on one stream, so no step
    counters are needed (scripts/halo_overhead.py times this path)."""

    def __init__(self, geometry, world, config=None, device=None, fused=False,
                 traversal="auto"):
        self.plan = SlabPlan(geometry, world)
        self.slabs = [SlabSolver(geometry, self.plan, r, config, device, traversal)
                      for r in range(world)]
        self.fused = bool(fused)
    def _exchange(self):
        for sl in self.slabs:
            r = sl.range
            if sl.send_up is not None:
                self.slabs[r.upper].recv_lo.copy_(sl.send_up)
            if sl.send_down is not None:
                self.slabs[r.lower].recv_hi.copy_(sl.send_down)

    def exchange_current(self):
        for sl in self.slabs:
            sl.pack(current=True)
        self._exchange()
        for sl in self.slabs:
            sl.unpack(current=True)

    def step(self, n=1, check=True):
        for _ in range(int(n)):
            if self.fused:
                # each slab: interior on the main stream, boundary layers on
                # its side stream after the neighbours' previous boundary
                # launches (they read the ghost tiles this step writes and
                # wrote the ghost tiles this step reads) -- the ordering the
                # IPC path gets from the step counters
                evs = [sl.last_boundary_event() for sl in self.slabs]
                for sl in self.slabs:
                    r = sl.range
                    waits = [evs[k] for k in (r.lower, r.upper) if k >= 0 and evs[k] is not None]
                    sl.step_overlapped(before=lambda sl=sl: self._arm(sl),
                                       after=lambda sl=sl: self._disarm(sl),
                                       wait_events=waits)
                for sl in self.slabs:
                    sl.finish()
                continue
            for sl in self.slabs:
                sl.step_boundary()
                sl.pack()
            self._exchange()
            for sl in self.slabs:
                sl.step_interior()
                sl.unpack()
                sl.finish()
        for sl in self.slabs:
            sl.join()
        if check:
            for sl in self.slabs:
                sl.solver.check()

    @staticmethod
    def _disarm(sl):
        a = sl.solver._args
        a.halo_up = a.halo_down = None

    def _arm(self, sl):
        """Point a slab's halo fields at its neighbours' ghost tiles of the
        copy this step writes (IpcHalo.arm with device pointers)."""
        a, r = sl.solver._args, sl.range
        dst = 1 - sl.solver.parity
        tile_bytes = 19 * 64 * sl.solver.store.flat.element_size()
        if r.upper >= 0:
            u = self.slabs[r.upper]
            a.halo_up = u.solver.store.copy_tensor(dst).data_ptr()
            if sl.compact:
                a.halo_up_cbase = u.ghost_cbase("lo").data_ptr()
            else:
                a.halo_up += u.ghost_lo[0] * tile_bytes
            a.halo_up_begin, a.halo_up_end = sl.top
        if r.lower >= 0:
            lo = self.slabs[r.lower]
            a.halo_down = lo.solver.store.copy_tensor(dst).data_ptr()
            if sl.compact:
                a.halo_down_cbase = lo.ghost_cbase("hi").data_ptr()
            else:
                a.halo_down += lo.ghost_hi[0] * tile_bytes
            a.halo_down_begin, a.halo_down_end = sl.bottom

    def fields_owned(self):
        return torch.cat([sl.fields_owned() for sl in self.slabs], dim=1)


class SlabWorkload(DistributedSlabRunner):
    """One rank of a bench run on any geometry: the slab of ``geometry``
    this rank owns, started from the perturbed equilibrium of
    workloads.perturbed_fields (seeded per rank) with its ghosts filled."""

    def __init__(self, geometry, world, rank, precision="f64", table="b200", device=None,
                 transport="nccl", arithmetic="reference", u0=(0.0, 0.0, 0.02),
                 storage="blocks", u_max_guard=0.05):
        from . import workloads
        if storage != "blocks":
            table = None
        cfg = SimulationConfig(tau=workloads.TAU, precision=precision, table=table,
                               arithmetic=arithmetic, storage=storage, u_max_guard=u_max_guard)
        super().__init__(geometry, world, rank, cfg, device, transport)
        s = self.slab.solver
        rho, u = workloads.perturbed_fields(s.t_n, s.store.tdtype, s.device, u0,
                                            seed=1234 + rank)
        s.init_from_macroscopic(rho, u)
        self.exchange_current()

    def halo_bytes_per_step(self):
        """Bytes this rank sends per step (80 values per boundary tile and
        direction of travel); it receives as many."""
        sl = self.slab
        n = sum(b.numel() for b in (sl.send_up, sl.send_down) if b is not None)
        return n * sl.solver.store.flat.element_size()


class SlabChannel(SlabWorkload):
    """The config-2 channel for N ranks: n^2 cross-section periodic along z,
    n * N long, one n^3 slab per rank (weak scaling)."""

    def __init__(self, n, world, rank, precision="f64", table="b200", device=None,
                 transport="nccl", arithmetic="reference", u0=(0.0, 0.0, 0.02)):
        from . import workloads
        super().__init__(workloads.channel_z(n, n * world), world, rank, precision, table,
                         device, transport, arithmetic, u0)


def plan_run(geometry, world, precision="f64", storage="blocks", budget_gb=179.0):
    """Host-only sizing of an N-GPU run (no device needed): per rank the z
    range, tiles (owned + ghost), non-solid nodes, bytes of fields and
    metadata, halo bytes per step, and whether it fits ``budget_gb``.
    Field bytes: 2 copies x 19 values per slot (blocks) or per non-solid
    node (compact); metadata 364 B per tile (node words + neighbour row),
    plus 76 B per tile for compact storage."""
    from .solver import SimulationConfig
    cfg = SimulationConfig(precision=precision, storage=storage)
    if cfg.storage == "auto":
        cfg = resolve_auto_storage_global(cfg, geometry)
    n_d = 8 if precision == "f64" else 4
    plan = SlabPlan(geometry, world)
    ranks = []
    for r in range(world):
        t = np.asarray(plan.local_types(geometry.types, r) if world > 1 else geometry.types) != 0
        mesh = tuple(-(-n // TILE) for n in t.shape)
        occ = np.zeros(tuple(m * TILE for m in mesh), dtype=bool)
        occ[:t.shape[0], :t.shape[1], :t.shape[2]] = t
        per_tile = occ.reshape(mesh[0], TILE, mesh[1], TILE, mesh[2], TILE).sum(axis=(1, 3, 5))
        t_n, n_fn = int((per_tile > 0).sum()), int(t.sum())
        rg = plan.ranges[r]
        layer = lambda z0: int((per_tile[:, :, z0] > 0).sum())   # noqa: E731
        halo_tiles = (layer(mesh[2] - 2) if rg.upper >= 0 else 0) + \
                     (layer(1 if rg.lower >= 0 else 0) if rg.lower >= 0 else 0)
        fields = 2 * 19 * n_d * (n_fn if cfg.storage == "compact" else 64 * t_n)
        meta = t_n * (364 + (76 if cfg.storage == "compact" else 0))
        ranks.append({"rank": r, "z": [rg.z0, rg.z1], "tiles": t_n, "nonsolid_nodes": n_fn,
                      "field_gb": round(fields / 1e9, 3), "metadata_gb": round(meta / 1e9, 3),
                      "halo_bytes_sent_received_per_step": 2 * 80 * n_d * halo_tiles,
                      "fits": (fields + meta) / 1e9 < budget_gb})
    return {"world": world, "precision": precision, "storage": cfg.storage,
            "table": cfg.table.value, "budget_gb": budget_gb, "ranks": ranks,
            "fits": all(r["fits"] for r in ranks)}

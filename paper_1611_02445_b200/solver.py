"""Solver: init, step and run of the tiled D3Q19 LBGK path on one GPU.

The reference defines this module only in its SPEC (the
step semantics are restated in SURVEY Appendix A).  API:

``SimulationConfig``  SPEC.md:335-340 (collision, fluid, tau > 0.5,
                      mrt_relaxation, precision f32|f64, u_max_guard=0.05),
                      plus ``table`` (default LayoutTable.B200) and
                      ``arithmetic``: "reference" (default; numpy's
                      unfused operation order, bit-identical to the
                      reference) or "fma" (fused multiply-adds in the
                      collision: fewer instructions, parity within the
                      stated 1e-12 tolerance; f64 only), and ``storage``:
                      "blocks" (default, the paper's 64-slot blocks) or
                      "compact" (only the non-solid slots of every block;
                      less DRAM traffic on sparse geometries)
                      or "auto" (compact, with the node-parallel step, when
                      the tile utilisation eta_t < AUTO_COMPACT_ETA of the
                      precision, else blocks).
``SimulationState``   SPEC.md:341-345 (geometry, tile grid, field store,
                      iteration, parity).
``Solver``            owns the device state; ``step(n)``, ``run(n)``,
                      ``macroscopic()``, ``fields_canonical()``.
``step(state)`` / ``run(config, geometry, iterations, outputs)``  SPEC ops.

Each step is one launch of the fused kernel (csrc/step.cu) reading copy
``parity`` and writing copy ``1 - parity`` (A/B buffers);
no host synchronisation happens between steps.  Divergence (NaN, or rho <= 0
in the quasi-compressible model) and the |u| guard are OR-ed by the kernel
into a per-iteration status word of a ring buffer; ``check()`` reads it and
raises ``DivergenceError`` with the exact iteration.
"""

import hashlib
import json
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .collision import CollisionModel, DivergenceError, FluidModel, fluid_code
from .geometry import Geometry
from .layout import TABLE_CODE, CompactFieldStore, FieldStore, LayoutTable
from .lattice import Q, WEIGHTS
from .tiling import DeviceTiling

STATUS_RING = 4096
GRAPH_STEPS = 64      # steps per captured CUDA graph (even: the parity is restored)
GRAPH_AUTO_TILES = 65536    # run(graph="auto"): replay graphs up to this many tiles


class CompressibilityWarning(UserWarning):
    """|u| exceeded SimulationConfig.u_max_guard."""


@dataclass
class SimulationConfig:
    collision: CollisionModel = CollisionModel.LBGK
    fluid: FluidModel = FluidModel.INCOMPRESSIBLE
    tau: float = 0.6
    mrt_relaxation: tuple = None
    precision: str = "f64"
    u_max_guard: float = 0.05
    table: LayoutTable = None      # default: B200 (blocks storage), XYZ (compact)
    mrt_matrix: object = None      # optional explicit 19x19 operator (overrides rates)
    arithmetic: str = "reference"  # "reference" (bit-exact) | "fma"
    storage: str = "blocks"        # "blocks" (the paper's 64-slot blocks) | "compact" | "auto"

    def __post_init__(self):
        self.collision = CollisionModel(getattr(self.collision, "value", self.collision))
        self.fluid = FluidModel(getattr(self.fluid, "value", self.fluid))
        if self.storage not in ("blocks", "compact", "auto"):
            raise ValueError(f"unknown storage: {self.storage!r}")
        if self.table is None and self.storage != "auto":
            self.table = LayoutTable.XYZ if self.storage == "compact" else LayoutTable.B200
        if self.table is not None:
            self.table = LayoutTable(getattr(self.table, "value", self.table))
        if not float(self.tau) > 0.5:
            raise ValueError(f"relaxation time must exceed 0.5: {self.tau}")
        if self.precision not in ("f32", "f64"):
            raise ValueError(f"unknown precision: {self.precision!r}")
        if self.arithmetic not in ("reference", "fma"):
            raise ValueError(f"unknown arithmetic: {self.arithmetic!r}")
        if self.storage == "auto" and self.table is not None:
            raise ValueError("storage='auto' picks the layout table itself; leave table unset")
        if self.storage == "compact" and self.table is not LayoutTable.XYZ:
            raise ValueError("compact storage keeps blocks in XYZ order: table must be xyz")
        if self.arithmetic == "fma" and self.precision != "f64":
            raise ValueError("arithmetic='fma' is f64-only: in f32 it drifts past the 1e-5 "
                             "parity bar (u: 1.1e-5 after 1000 cavity-64 steps)")
        if self.collision is CollisionModel.MRT:
            from .collision import default_mrt_rates
            rates = (default_mrt_rates(self.tau) if self.mrt_relaxation is None
                     else np.asarray(self.mrt_relaxation, dtype=np.float64))
            if rates.shape != (19,):
                raise ValueError("mrt_relaxation needs 19 moment rates")
            self.mrt_relaxation = tuple(float(r) for r in rates)

    @property
    def mrt_operator(self):
        """float64 M^-1 S M of the configured rates (None for LBGK)."""
        if self.collision is not CollisionModel.MRT:
            return None
        if self.mrt_matrix is not None:
            op = np.asarray(self.mrt_matrix, dtype=np.float64)
            if op.shape != (19, 19):
                raise ValueError("mrt_matrix must be 19x19")
            return op
        from .collision import mrt_operator
        return mrt_operator(self.mrt_relaxation, dtype=np.float64)

    @property
    def dtype(self):
        return np.float64 if self.precision == "f64" else np.float32


@dataclass
class SimulationState:
    geometry: Geometry
    tile_grid: object
    field_store: FieldStore
    iteration: int = 0
    parity: int = 0
    config: SimulationConfig = None
    solver: object = field(default=None, repr=False)


class Solver:
    """Device-resident tiled LBGK solver for one geometry on one GPU."""

    def __init__(self, geometry, config=None, device=None, tiling=None, index64=False,
                 traversal="auto", initial=(1.0, (0.0, 0.0, 0.0))):
        """``index64`` forces the step's 64-bit addressing path (used
        automatically when neighbour offsets exceed 32 bits, i.e. beyond
        ~1.76 M tiles); exposed for tests and measurements.

        ``traversal``: the order the step visits tiles in.  "tile" is the
        tile-list order (z outer).  "auto" switches fp32 block storage to a
        y-blocked order (traversal_order) when a z-layer of tiles moves more
        bytes than L2_REUSE_BUDGET, so that the 128-byte L2 lines a tile
        shares with its z neighbour are still resident when the neighbour
        runs (fp32 512^3: +2-3% in a same-box A/B).  fp64 blocks share no
        lines across z and lose DRAM streaming locality in the blocked order
        (0.974 -> 0.945), so they keep the tile order, as does compact
        storage (measured slower).  An int forces the
        blocking with that many tile rows.  "nodes" (compact storage only)
        runs the node-parallel step: one thread per non-solid node in store
        order instead of one per tile slot (csrc/step_compact.cuh:
        step_kernel_nodes); "auto" picks it for compact storage below tile
        utilisation AUTO_NODES_ETA.

        ``initial``: the uniform equilibrium (rho, (ux, uy, uz)) both copies
        start from (default the cold start rho 1, u 0)."""
        self.config = config if config is not None else SimulationConfig()
        self.geometry = geometry
        self.tiling = tiling if tiling is not None else DeviceTiling(geometry, device)
        self.device = self.tiling.device
        self.t_n = self.tiling.t_n
        self.n_fn = self.tiling.n_fn
        if self.config.storage == "auto":
            self.config = resolve_auto_storage(self.config, self.n_fn, self.t_n)
        if self.config.storage == "compact":
            self.store = CompactFieldStore(self.tiling, self.config.table, self.config.dtype)
        else:
            self.store = FieldStore(self.t_n, self.config.table, self.config.dtype, self.device,
                                    zero=False)
        self.code = self.store.code
        self.fluid = fluid_code(self.config.fluid)
        self.table = TABLE_CODE[self.config.table]
        self.iteration = 0
        self.parity = 0
        self._checked = 0
        self.guard_iterations = []
        self.status = torch.zeros(STATUS_RING, dtype=torch.int32, device=self.device)
        self._grid = None
        self._args = nat.StepArgs()
        a = self._args
        a.dtype, a.fluid, a.table, a.variant = self.code, self.fluid, self.table, nat.FULL
        a.t_n, a.tile_begin, a.tile_end = self.t_n, 0, self.t_n
        a.nbr = self.tiling.nbr.data_ptr()
        a.meta = self.tiling.meta.data_ptr()
        a.tau = float(self.config.tau)
        a.inlet_u[:] = list(geometry.inlet_velocity)
        a.outlet_rho = float(geometry.outlet_density)
        a.u_guard = float(self.config.u_max_guard or 0.0)
        a.rel32 = int(self.tiling.rel32 and not index64)
        a.arith = nat.ARITH_FMA if self.config.arithmetic == "fma" else nat.ARITH_REFERENCE
        if self.config.storage == "compact":
            # compact storage: rel32 means every element offset of a copy
            # fits 32 bits (the kernel's OFF32 path)
            a.rel32 = int(Q * self.n_fn < 2 ** 32 and not index64)
            a.cbase = self.store.base.data_ptr()
            a.cnf = self.store.nf.data_ptr()
            a.crank = self.store.rank.data_ptr()
        self._mrt_op = self.config.mrt_operator        # kept alive for the ABI pointer
        if self._mrt_op is not None:
            self._mrt_op = np.ascontiguousarray(self._mrt_op)
            a.collision = nat.MRT
            a.mrt_op = self._mrt_op.ctypes.data
        else:
            a.collision = nat.LBGK
        self._copies = (self.store.copy_tensor(0).data_ptr(), self.store.copy_tensor(1).data_ptr())
        self.nodes = None
        if use_nodes(self.config, self.n_fn, self.t_n, traversal):
            if not a.rel32:
                raise ValueError("the node-parallel step needs 32-bit offsets "
                                 "(19 * n_fn < 2^32)")
            self.nodes = self.store.node_records(self.tiling)
            a.node_meta = self.nodes["node_meta"].data_ptr()
            a.node_rec = self.nodes["node_rec"].data_ptr()
            a.unit_tile = self.nodes["unit_tile"].data_ptr()
            a.entries = self.nodes["entries"].data_ptr()
            a.node_begin, a.node_end = 0, self.n_fn
            traversal = "tile"
        self.order = traversal_order(self.tiling, self.store, traversal)
        a.order = self.order.data_ptr() if self.order is not None else None
        self._graphs = {}
        self._iter_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._iter_dev_value = 0
        # the cold start (rho 1, u 0) or the uniform
        # equilibrium `initial` = (rho, u), written once into both copies
        self.init_equilibrium(float(initial[0]), tuple(float(v) for v in initial[1]))

    # -- initial state -------------------------------------------------------
    def init_equilibrium(self, rho=1.0, u=(0.0, 0.0, 0.0)):
        """Both copies, all 64 slots of every tile := equilibrium(rho, u)
        (the conventional cold start uses rho=1, u=0)."""
        nat.require_cuda(self.device)
        for c in (0, 1):
            blk = self._blocks_out(c)
            nat.call("tlbm_init_equilibrium", nat.ptr(blk), self.code,
                     self.fluid, self.table, self.t_n, float(rho), *(float(v) for v in u),
                     nat.stream_ptr(self.device))
            self._blocks_in(c, blk)
        self._reset_counters()

    # the paper-layout blocks of one copy for the block-store kernels (init,
    # readout): the copy itself, or an expanded temporary for compact storage
    def _blocks_out(self, c, current=False):
        if isinstance(self.store, CompactFieldStore):
            if current:
                return self.store.to_blocks(c)
            return torch.empty(self.t_n * Q * 64, dtype=self.store.tdtype, device=self.device)
        return self.store.copy_tensor(c)

    def _blocks_in(self, c, blk):
        if isinstance(self.store, CompactFieldStore):
            self.store.from_blocks(c, blk)

    def init_from_macroscopic(self, rho, u):
        """Both copies := equilibrium(rho, u) per slot; rho (t_n, 64), u
        (3, t_n, 64) canonical arrays (numpy or CUDA tensors)."""
        nat.require_cuda(self.device)
        dt = self.store.tdtype
        r = torch.as_tensor(rho).to(self.device, dt).contiguous()
        v = torch.as_tensor(u).to(self.device, dt).contiguous()
        if tuple(r.shape) != (self.t_n, 64) or tuple(v.shape) != (3, self.t_n, 64):
            raise ValueError("expected rho (t_n, 64) and u (3, t_n, 64)")
        for c in (0, 1):
            blk = self._blocks_out(c)
            nat.call("tlbm_init_from_macroscopic", nat.ptr(blk),
                     self.code, self.fluid, self.table, self.t_n, nat.ptr(r), nat.ptr(v),
                     nat.stream_ptr(self.device))
            self._blocks_in(c, blk)
        self._reset_counters()

    def set_fields_canonical(self, values, copy=None):
        """Overwrite a copy (default: both) from (19, t_n, 64) canonical values."""
        for c in ((0, 1) if copy is None else (copy,)):
            self.store.fill_canonical(c, values)

    def _reset_counters(self):
        self.iteration = 0
        self.parity = 0
        self._checked = 0
        self.guard_iterations = []
        self.status.zero_()

    # -- stepping ------------------------------------------------------------
    def step(self, n=1, variant=nat.FULL, check=True, graph=False):
        """Advance n iterations (no host sync unless ``check`` and the status
        ring is full or n is exhausted).  ``graph``: run whole blocks of
        GRAPH_STEPS iterations as replays of a captured CUDA graph (one
        launch per block instead of one ctypes call per step; for small
        domains whose step takes a few microseconds)."""
        nat.require_cuda(self.device)
        n = int(n)
        if graph:
            while n >= GRAPH_STEPS:
                if self.iteration + GRAPH_STEPS - self._checked > STATUS_RING:
                    self.check()
                self._replay(int(variant))
                n -= GRAPH_STEPS
        a = self._args
        a.variant = int(variant)
        a.tile_begin, a.tile_end = 0, self.t_n
        a.node_begin, a.node_end = 0, self.n_fn
        a.iter_counter = None
        stream = nat.stream_ptr(self.device)
        lib = nat.load()
        base = self.status.data_ptr()
        for _ in range(n):
            if self.iteration - self._checked >= STATUS_RING:
                self.check()
            a.f_src = self._copies[self.parity]
            a.f_dst = self._copies[1 - self.parity]
            a.flags = base + 4 * (self.iteration % STATUS_RING)
            rc = lib.tlbm_step(nat.ctypes.byref(a), stream)
            if rc:
                nat.check(rc)
            self.parity ^= 1
            self.iteration += 1
        if check:
            self.check()
        return self

    def _replay(self, variant):
        """GRAPH_STEPS iterations as one CUDA graph replay.  The graph holds
        GRAPH_STEPS step launches (copies alternating from the current
        parity, status slot (device iteration counter + i) % STATUS_RING)
        and a last node advancing the device counter, so it replays without
        host-side parameter updates."""
        key = (self.parity, variant)
        g = self._graphs.get(key)
        if g is None:
            g = self._capture(variant)
            self._graphs[key] = g
        if self._iter_dev_value != self.iteration:
            self._iter_dev.fill_(self.iteration)
        g.replay()
        self.iteration += GRAPH_STEPS
        self._iter_dev_value = self.iteration

    def _capture(self, variant):
        a = nat.StepArgs()
        ctypes_copy = nat.ctypes.pointer(a)
        nat.ctypes.memmove(ctypes_copy, nat.ctypes.byref(self._args), nat.ctypes.sizeof(a))
        a.variant = variant
        a.tile_begin, a.tile_end = 0, self.t_n
        a.node_begin, a.node_end = 0, self.n_fn
        a.flags = self.status.data_ptr()
        a.iter_counter = self._iter_dev.data_ptr()
        a.ring_len = STATUS_RING
        lib = nat.load()
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize(self.device)
        with torch.cuda.device(self.device), torch.cuda.graph(g):
            stream = nat.stream_ptr(self.device)
            par = self.parity
            for i in range(GRAPH_STEPS):
                a.f_src, a.f_dst = self._copies[par], self._copies[1 - par]
                a.iter_add = i
                nat.check(lib.tlbm_step(nat.ctypes.byref(a), stream))
                par ^= 1
            nat.check(lib.tlbm_advance_counter(nat.ptr(self._iter_dev), GRAPH_STEPS, stream))
        return g

    def check(self):
        """Read the status ring; raise DivergenceError at the first divergent
        iteration, record |u| guard trips (CompressibilityWarning)."""
        pending = self.iteration - self._checked
        if pending <= 0:
            return
        st = self.status.cpu().numpy()
        for it in range(self._checked, self.iteration):
            w = int(st[it % STATUS_RING])
            if w & nat.FLAG_GUARD:
                self.guard_iterations.append(it)
            if w & nat.FLAG_DIVERGED:
                self.status.zero_()
                self._checked = self.iteration
                raise DivergenceError("simulation diverged (NaN or non-positive density)",
                                      iteration=it)
        if st.any():
            self.status.zero_()
        if self.guard_iterations and self.guard_iterations[-1] >= self._checked:
            warnings.warn(f"|u| exceeded u_max_guard={self.config.u_max_guard} at iteration "
                          f"{self.guard_iterations[-1]}", CompressibilityWarning, stacklevel=2)
        self._checked = self.iteration

    def run(self, iterations, check_every=STATUS_RING, graph="auto"):
        """``iterations`` steps, the status ring checked every ``check_every``.
        ``graph="auto"`` replays CUDA graphs when a step is short enough for
        the per-launch cost to show (t_n <= GRAPH_AUTO_TILES; cavity 64^3:
        16.4 -> 13.3 us per step); True / False force it."""
        if graph == "auto":
            graph = 0 < self.t_n <= GRAPH_AUTO_TILES
        left = int(iterations)
        while left > 0:
            k = min(left, check_every)
            self.step(k, check=True, graph=graph)
            left -= k
        return self

    # -- readout -------------------------------------------------------------
    def macroscopic(self, device=False, copy=None):
        """(rho (t_n,64), u (3,t_n,64), p (t_n,64)) of the current copy, in
        canonical slot order (collision.py:75-91 on read_canonical)."""
        nat.require_cuda(self.device)
        c = self.parity if copy is None else copy
        dt = self.store.tdtype
        rho = torch.empty((self.t_n, 64), dtype=dt, device=self.device)
        u = torch.empty((3, self.t_n, 64), dtype=dt, device=self.device)
        p = torch.empty((self.t_n, 64), dtype=dt, device=self.device)
        flags = torch.zeros(1, dtype=torch.int32, device=self.device)
        nat.call("tlbm_macroscopic", nat.ptr(self._blocks_out(c, current=True)), self.code,
                 self.fluid,
                 self.table, self.t_n, nat.ptr(rho), nat.ptr(u), nat.ptr(p), nat.ptr(flags),
                 nat.stream_ptr(self.device))
        if self.fluid == nat.QUASI and int(flags.item()) & nat.FLAG_DIVERGED:
            raise DivergenceError("non-positive density in quasi-compressible flow",
                                  iteration=self.iteration)
        if device:
            return rho, u, p
        return rho.cpu().numpy(), u.cpu().numpy(), p.cpu().numpy()

    def fields_canonical(self, copy=None, device=False):
        """(19, t_n, 64) canonical populations of the current (or given) copy."""
        return self.store.read_canonical(self.parity if copy is None else copy, device=device)

    @property
    def tile_grid(self):
        if self._grid is None:
            self._grid = self.tiling.grid()
        return self._grid

    def nonsolid_mask(self, device=False):
        m = (self.tiling.meta & 1).bool()
        return m if device else m.cpu().numpy()

    def total_mass(self):
        """Sum of rho over non-solid slots (fp64 accumulation on the GPU)."""
        rho, _, _ = self.macroscopic(device=True)
        return float(rho[self.nonsolid_mask(device=True)].double().sum().item())

    def to_dense(self, canonical):
        """Scatter a (..., t_n, 64) canonical array to (..., nx, ny, nz) on the
        GPU (absent tiles / padding dropped; absent tiles read as 0)."""
        x = torch.as_tensor(canonical, device=self.device)
        lead = tuple(x.shape[:-2])
        pd = tuple(m * 4 for m in self.tiling.mesh)
        out = torch.zeros(lead + pd, dtype=x.dtype, device=self.device)
        ne = self.tiling.non_empty.long()
        s = torch.arange(64, device=self.device)
        xi = ne[:, 0:1] + (s & 3)
        yi = ne[:, 1:2] + ((s >> 2) & 3)
        zi = ne[:, 2:3] + (s >> 4)
        out[..., xi, yi, zi] = x
        nx, ny, nz = self.tiling.dims
        return out[..., :nx, :ny, :nz]

    # -- checkpoint / resume --------------------------------------------------
    def save_checkpoint(self, path):
        """Write the current state to ``path`` (.npz): the canonical
        (19, t_n, 64) populations of the current copy in the working dtype,
        the iteration, the configuration and a fingerprint of the geometry.
        Only the current copy is state: the next step rewrites every active
        slot of the other one, and solid slots are never read."""
        self.check()
        cfg = {k: (v.value if hasattr(v, "value") else v)
               for k, v in self.config.__dict__.items() if k != "mrt_matrix"}
        extra = {}
        if self.config.mrt_matrix is not None:
            extra["mrt_matrix"] = np.asarray(self.config.mrt_matrix, dtype=np.float64)
        np.savez(path, format=np.array(CHECKPOINT_FORMAT), f=self.fields_canonical(),
                 iteration=np.int64(self.iteration), config=np.array(json.dumps(cfg)),
                 geometry=np.array(geometry_fingerprint(self.geometry)), **extra)

    def load_checkpoint(self, path):
        """Restore a state written by save_checkpoint into this solver (same
        geometry and precision); stepping on is bit-identical to never having
        stopped."""
        with np.load(path, allow_pickle=False) as z:
            if str(z["format"]) != CHECKPOINT_FORMAT:
                raise ValueError(f"{path}: not a {CHECKPOINT_FORMAT} checkpoint")
            if str(z["geometry"]) != geometry_fingerprint(self.geometry):
                raise ValueError(f"{path}: checkpoint was written for another geometry")
            f = z["f"]
            if f.dtype != self.config.dtype or f.shape != (Q, self.t_n, 64):
                raise ValueError(f"{path}: fields {f.dtype} {f.shape} do not fit this solver "
                                 f"({np.dtype(self.config.dtype)}, t_n {self.t_n})")
            it = int(z["iteration"])
        self._reset_counters()
        self.iteration = self._checked = it
        self.parity = it & 1
        self.store.fill_canonical(self.parity, f)
        return self

    @property
    def state(self):
        return SimulationState(self.geometry, self.tile_grid, self.store, self.iteration,
                               self.parity, self.config, self)


def init_state(config, geometry, device=None):
    """Solver init: tiling, two-copy store, equilibrium start."""
    return Solver(geometry, config, device).state


def step(state):
    """One LBM iteration; returns the updated state."""
    s = state.solver
    if s is None:
        raise ValueError("state has no solver attached; build it with init_state()")
    s.step(1)
    state.iteration, state.parity = s.iteration, s.parity
    return state


def run(config, geometry, iterations, outputs=None, device=None, check_every=STATUS_RING,
        resume_from=None, graph="auto"):
    """Iterate ``iterations`` steps; returns (state,
    diagnostics).

    ``outputs``: a callable(solver) run at the end, or a dict with any of
      "convergence_every": k   relative L2 change of u every k steps
      "tolerance": eps         stop early once that change is below eps
      "vtk": path, "csv": path write the final rho/u (legacy VTK / CSV slice)
      "checkpoint": path       save the final state (Solver.save_checkpoint)
    Zero iterations return the initial state unchanged.
    ``resume_from``: a checkpoint path; ``iterations`` more steps are run from
    it.  ``graph``: replay CUDA graphs of GRAPH_STEPS steps (Solver.step).
    """
    from .output import ConvergenceEstimator, dense_macroscopic, write_csv_slice, write_vtk
    solver = (Solver(geometry, config, device) if resume_from is None
              else resume(resume_from, geometry, config, device))
    opts = outputs if isinstance(outputs, dict) else {}
    every = int(opts.get("convergence_every") or 0)
    tol = opts.get("tolerance")
    est = ConvergenceEstimator(solver, every) if every > 0 else None
    if est is not None:
        est()
    left = int(iterations)
    converged = False
    while left > 0:
        k = min(left, every if every > 0 else check_every)
        solver.run(k, check_every=check_every, graph=graph)
        left -= k
        if est is not None:
            change = est()
            if tol is not None and change is not None and change < tol:
                converged = True
                break
    diagnostics = {"iterations": solver.iteration, "t_n": solver.t_n, "n_fn": solver.n_fn,
                   "guard_iterations": list(solver.guard_iterations),
                   "convergence": list(est.history) if est is not None else [],
                   "converged": converged}
    if opts.get("checkpoint"):
        solver.save_checkpoint(opts["checkpoint"])
    if opts.get("vtk") or opts.get("csv"):
        rho, u = dense_macroscopic(solver)
        if opts.get("vtk"):
            write_vtk(opts["vtk"], rho, u)
        if opts.get("csv"):
            write_csv_slice(opts["csv"], rho, u)
    if callable(outputs):
        outputs(solver)
    return solver.state, diagnostics


L2_REUSE_BUDGET = 40 << 20    # bytes of step traffic between a tile and its z neighbour


def traversal_order(tiling, store, traversal="auto"):
    """Tile visiting order of the step (tlbm_step_args.order), or None for
    the tile-list order.

    The tile list is z outer, so a tile's z neighbour comes a whole layer of
    tiles later.  Lines the two share (a 128-byte L2 line holds two fp32
    z-planes of a block; compact blocks are not line aligned) are fetched
    twice once a layer's traffic exceeds what L2 keeps.  The blocked order
    visits the tiles in bands of ``yb`` tile rows, z inside a band: a z
    neighbour is then ``yb`` rows away and a y neighbour one row, except
    across band edges."""
    if traversal == "tile" or tiling.t_n == 0:
        return None
    if traversal == "auto" and (store.flat.element_size() != 4
                                or isinstance(store, CompactFieldStore)):
        return None
    ntx, nty, ntz = tiling.mesh
    n_d = store.flat.element_size()
    per_tile = 2.0 * store.flat.numel() / 2 / max(tiling.t_n, 1) * n_d   # read + write
    coords = tiling.non_empty.to(torch.int64) // 4
    if isinstance(traversal, int):
        yb = max(1, int(traversal))
    else:
        layers = int(torch.unique(coords[:, 2]).numel())
        rows = int(torch.unique(coords[:, 1] * ntz + coords[:, 2]).numel())
        layer_bytes = tiling.t_n / max(layers, 1) * per_tile
        if layer_bytes <= L2_REUSE_BUDGET:
            return None
        row_bytes = tiling.t_n / max(rows, 1) * per_tile
        yb = max(1, int(L2_REUSE_BUDGET // max(row_bytes, 1.0)))
        if yb >= nty:
            return None
    tx, ty, tz = coords[:, 0], coords[:, 1], coords[:, 2]
    key = (((ty // yb) * ntz + tz) * nty + ty) * ntx + tx
    return torch.argsort(key, stable=True).to(torch.int32)


# traversal="auto" on compact storage: the node-parallel step below this
# tile utilisation.  From the bench porosity block (profiles/r2b_bench_n1.json):
# nodes beats the tile-parallel compact kernel at every porosity up to 0.8
# (fp64 0.879 vs 0.749 BU at porosity 0.2, fp32 0.714 vs 0.538) and trails
# it slightly on near-full tiles (fp64 0.886 vs 0.895 at eta_t 0.971).
AUTO_NODES_ETA = 0.95


def use_nodes(config, n_fn, t_n, traversal):
    """Does a solver with this configuration run the node-parallel step?"""
    if traversal == "nodes":
        if config.storage != "compact":
            raise ValueError("traversal='nodes' needs storage='compact'")
        return True
    if traversal != "auto" or config.storage != "compact" or not t_n:
        return False
    # the node-parallel step addresses a copy with 32-bit offsets
    return n_fn / (64.0 * t_n) < AUTO_NODES_ETA and Q * n_fn < 2 ** 32


# storage="auto": compact storage (with the node-parallel step) below this
# tile utilisation, per precision.  From the bench porosity block
# (profiles/r2b_bench_n1.json), nodes vs the paper's blocks: fp64 +42% at
# eta_t 0.658 (porosity 0.2), +7% at 0.866 (0.6), +0.5% at 0.904 (0.7), +2%
# on the vessel tree (0.927), -5% at 0.939 (0.8); fp32 +31% at 0.658, tie
# at 0.825 (0.5), -5% at 0.866.
AUTO_COMPACT_ETA = {"f64": 0.93, "f32": 0.83}


def resolve_auto_storage(config, n_fn, t_n):
    """The concrete configuration storage="auto" stands for on a tiling."""
    import dataclasses
    eta = n_fn / (64.0 * t_n) if t_n else 1.0
    compact = eta < AUTO_COMPACT_ETA[config.precision]
    return dataclasses.replace(config, storage="compact" if compact else "blocks", table=None)


CHECKPOINT_FORMAT = "tlbm-checkpoint-1"


def geometry_fingerprint(geometry):
    """sha256 over the voxel tags, shape, boundary values and periodic flags."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(geometry.types, dtype=np.uint8).tobytes())
    h.update(json.dumps([list(geometry.shape), [float(v) for v in geometry.inlet_velocity],
                         float(geometry.outlet_density),
                         [bool(p) for p in geometry.periodic]]).encode())
    return h.hexdigest()


def resume(path, geometry, config=None, device=None):
    """A Solver restored from a checkpoint; ``config`` defaults to the one
    stored in the checkpoint."""
    if config is None:
        with np.load(path, allow_pickle=False) as z:
            kw = json.loads(str(z["config"]))
            if "mrt_matrix" in z.files:
                kw["mrt_matrix"] = z["mrt_matrix"]
        if kw.get("mrt_relaxation") is not None:
            kw["mrt_relaxation"] = tuple(kw["mrt_relaxation"])
        config = SimulationConfig(**kw)
    return Solver(geometry, config, device).load_checkpoint(path)


def rest_weights(dtype=np.float64):
    return WEIGHTS.astype(dtype)

"""Device tiler: Alg. 1 behind the reference's tiling API.

``build_tiling(geometry)`` uploads the voxel tags once and runs libtlbm's
tiler kernels (csrc/tiler.cu): tile occupancy, an order-stable compaction in
(z outer, y, x inner) scan order, the corner list, the 27-delta neighbour-tile
map and the per-slot node metadata the step reads.  The returned ``TileGrid``
has the reference's fields and values (tiling.py:19-83) bit for bit; the
device-resident arrays stay attached as ``grid.device`` so the solver does
not rebuild them.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as nat
from .geometry import Geometry

TILE = 4


@dataclass
class TileGrid:
    a: int
    dims: tuple
    padded_dims: tuple
    tile_map: np.ndarray
    non_empty: np.ndarray
    device: object = field(default=None, repr=False, compare=False)

    @property
    def t_n(self):
        return int(self.non_empty.shape[0])

    @property
    def nodes_per_tile(self):
        return self.a ** 3

    @property
    def mesh_shape(self):
        return self.tile_map.shape


@dataclass
class TileStats:
    t_n: int
    n_fn: int
    eta_t: float
    n_tfn: float
    n_tsn: float
    eta_f: float
    eta_e: float


def periodic_mask(periodic):
    return sum(1 << a for a in range(3) if periodic[a])


class DeviceTiling:
    """Tile structures of one geometry resident on one GPU.

    tile_map  (ntx, nty, ntz) int32     -1 for empty tiles
    non_empty (t_n, 3) int32            tile corners, scan order
    nbr       (t_n, 27) int32           neighbour tile per delta, -1 absent
    meta      (t_n, 64) uint32          per-slot node word (csrc/d3q19.cuh)
    counts    (t_n,) int32              non-solid nodes per tile

    The voxel tags go to the device only while the tiler runs (1 B/voxel, 2 GB
    at 2048 x 1024^2); afterwards the step needs only the per-tile arrays.
    """

    def __init__(self, geometry, device=None):
        if not isinstance(geometry, Geometry):
            raise TypeError("build_tiling expects a Geometry")
        self.device = nat.require_cuda(device)
        self.dims = tuple(int(v) for v in geometry.shape)
        self.periodic = tuple(geometry.periodic)
        nx, ny, nz = self.dims
        self.mesh = tuple(-(-n // TILE) for n in self.dims)
        stream = nat.stream_ptr(self.device)
        types = torch.from_numpy(geometry.types).to(self.device)
        self.tile_map = torch.empty(self.mesh, dtype=torch.int32, device=self.device)
        scratch = torch.empty(int(nat.load().tlbm_tiling_scratch_bytes(nx, ny, nz)),
                              dtype=torch.uint8, device=self.device)
        t_n = nat.c_i64(0)
        nat.call("tlbm_tile_map", nat.ptr(types), nx, ny, nz, nat.ptr(self.tile_map),
                 nat.ptr(scratch), nat.ctypes.byref(t_n), stream)
        del scratch
        self.t_n = int(t_n.value)
        t = max(self.t_n, 1)
        self.non_empty = torch.empty((t, 3), dtype=torch.int32, device=self.device)[:self.t_n]
        nat.call("tlbm_tile_list", nat.ptr(self.tile_map), *self.mesh, nat.ptr(self.non_empty),
                 self.t_n, stream)
        self.nbr = torch.empty((t, 27), dtype=torch.int32, device=self.device)[:self.t_n]
        nat.call("tlbm_tile_neighbors", nat.ptr(self.tile_map), *self.mesh,
                 nat.ptr(self.non_empty), self.t_n, periodic_mask(self.periodic),
                 nat.ptr(self.nbr), stream)
        self.meta = torch.empty((t, 64), dtype=torch.int32, device=self.device)[:self.t_n]
        bad = torch.zeros(2, dtype=torch.int32, device=self.device)
        nat.call("tlbm_node_meta", nat.ptr(types), nx, ny, nz,
                 periodic_mask(self.periodic), nat.ptr(self.non_empty), self.t_n,
                 nat.ptr(self.meta), nat.ptr(bad), stream)
        del types           # stream-ordered: the caching allocator reuses it after meta
        self.counts = torch.empty(t, dtype=torch.int32, device=self.device)[:self.t_n]
        nat.call("tlbm_tile_counts", nat.ptr(self.meta), self.t_n, nat.ptr(self.counts), stream)
        n_bad_face, n_bad_tag = (int(v) for v in bad.cpu())
        if n_bad_tag:
            raise ValueError(f"{n_bad_tag} voxels carry unknown node type tags")
        if n_bad_face:
            raise ValueError(f"{n_bad_face} inlet/outlet nodes do not lie on exactly one "
                             "axis-aligned domain face")
        self.n_fn = int(self.counts.sum().item()) if self.t_n else 0
        self.rel32 = self._offsets_fit_int32()

    def _offsets_fit_int32(self, chunk=1 << 20):
        """True if every neighbour is within 2^31 values of its tile in the
        store (|nbr - t| * 19 * 64 < 2^31), enabling the step kernel's 32-bit
        relative addressing."""
        limit = (2 ** 31 - 1) // (19 * 64) - 1
        for b in range(0, self.t_n, chunk):
            blk = self.nbr[b:b + chunk]
            t = torch.arange(b, b + blk.shape[0], device=self.device, dtype=torch.int32)
            d = torch.where(blk >= 0, (blk - t[:, None]).abs(), torch.zeros_like(blk))
            if int(d.max().item()) > limit:
                return False
        return True

    def grid(self):
        return TileGrid(a=TILE, dims=self.dims,
                        padded_dims=tuple(m * TILE for m in self.mesh),
                        tile_map=self.tile_map.cpu().numpy(),
                        non_empty=self.non_empty.cpu().numpy(), device=self)


def build_tiling(geometry, a=4):
    """Alg. 1 on the GPU; same result as tiling.py:51-83 (a must be 4, the
    solver tile edge, SPEC.md tiling: "4 is the supported solver size")."""
    if int(a) != TILE:
        raise ValueError(f"the B200 tiler builds the solver's a = 4 tiling, got a = {a}")
    return DeviceTiling(geometry).grid()


def _device_of(grid, geometry):
    if grid.device is not None:
        return grid.device
    return DeviceTiling(geometry)


def faces_edges_per_tile(grid):
    """Common faces / edges per non-empty tile (tiling.py:86-117), on the GPU."""
    if grid.t_n == 0:
        raise ValueError("tile grid has no non-empty tiles")
    dev = nat.require_cuda()
    occ = torch.from_numpy(grid.tile_map).to(dev) >= 0
    faces = 0
    for axis in range(3):
        n = occ.shape[axis]
        faces += int((occ.narrow(axis, 0, n - 1) & occ.narrow(axis, 1, n - 1)).sum())
    edges = 0
    for a1, a2 in ((0, 1), (0, 2), (1, 2)):
        n1, n2 = occ.shape[a1] - 1, occ.shape[a2] - 1
        if n1 <= 0 or n2 <= 0:
            continue
        quad = None
        for d1, d2 in ((0, 0), (1, 0), (0, 1), (1, 1)):
            part = occ.narrow(a1, d1, n1).narrow(a2, d2, n2)
            quad = part if quad is None else quad & part
        edges += int(quad.sum())
    return faces / grid.t_n, edges / grid.t_n


def tile_utilization(grid, geometry):
    """TileStats by exact enumeration (tiling.py:120-138)."""
    if grid.t_n == 0:
        raise ValueError("geometry contains no non-solid nodes")
    dt = _device_of(grid, geometry)
    n_fn = dt.n_fn
    n_tn = grid.nodes_per_tile
    eta_f, eta_e = faces_edges_per_tile(grid)
    return TileStats(t_n=grid.t_n, n_fn=n_fn, eta_t=n_fn / (grid.t_n * n_tn),
                     n_tfn=n_fn / grid.t_n, n_tsn=n_tn - n_fn / grid.t_n,
                     eta_f=eta_f, eta_e=eta_e)


def per_tile_nonsolid_counts(grid, geometry):
    """Non-solid nodes per tile in tile order (tiling.py:141-152)."""
    return _device_of(grid, geometry).counts.cpu().numpy().astype(np.int64)


def overhead_generic(eta_t):
    """(1 - eta_t) / eta_t (tiling.py:155-159)."""
    if not 0.0 < eta_t <= 1.0:
        raise ValueError(f"tile utilization must be in (0, 1]: {eta_t}")
    return (1.0 - eta_t) / eta_t


def overhead_memory(eta_t, q=19, n_d=8, n_t=1):
    """Memory overhead vs the q*n_d B/node minimum (tiling.py:162-175)."""
    if not 0.0 < eta_t <= 1.0:
        raise ValueError(f"tile utilization must be in (0, 1]: {eta_t}")
    if q <= 0 or n_d <= 0 or n_t < 0:
        raise ValueError("q and n_d must be positive, n_t non-negative")
    return (2.0 * q * n_d + n_t) / (eta_t * q * n_d) - 1.0, (2.0 - eta_t) / eta_t


def channel_tiling_sweep(shape, d, axis=0, a=4):
    """Tile utilisation of the 16 transverse placements (off1, off2) of a
    straight channel (tiling.py:178-194): the cross-section repeats along the
    axis, so one a-long slab per placement gives the infinite channel's
    eta_t.  Returns ([((off1, off2), Fraction eta_t)], Fraction mean)."""
    from fractions import Fraction

    from .geometry import generate_channel
    if a != TILE:
        raise ValueError(f"only the solver tile edge {TILE} is supported, got {a}")
    out = []
    for off1, off2 in ((i, j) for i in range(a) for j in range(a)):
        g = generate_channel(shape, d, axis=axis, offsets=(off1, off2), length=a)
        grid = build_tiling(g, a)
        out.append(((off1, off2), Fraction(g.nonsolid_count(), grid.t_n * a ** 3)))
    return out, sum(e for _, e in out) / len(out)


def bu_propagation_estimate(eta_f, eta_e):
    """The paper's empirical bandwidth-utilisation fit of the gather
    (tiling.py:197-216; fitted on one GPU, for comparison only):
    0.92 - eta_f/14.28 - eta_e/25.74 + 0.00104/(2.9 - eta_f) + 0.0023/(2.81 - eta_e).
    Raises at the fit's poles eta_f = 2.9, eta_e = 2.81."""
    for v, pole, name in ((eta_f, 2.9, "eta_f"), (eta_e, 2.81, "eta_e")):
        if v == pole:
            raise ValueError(f"{name} = {pole} is a singularity of the fit")
    return (0.92 - eta_f / 14.28 - eta_e / 25.74
            + 0.00104 / (2.9 - eta_f) + 0.0023 / (2.81 - eta_e))


def edge_face_plane_residual(eta_f, eta_e):
    """eta_e - (1.85 eta_f - 2.56): distance from the paper's coarse
    edge/face relation (tiling.py:219-221)."""
    return eta_e - (1.85 * eta_f - 2.56)

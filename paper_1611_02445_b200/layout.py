"""Per-tile data-block layouts and the two-copy field store.

Mirrors ``tilelbm.layout`` (reference layout.py:28-167): one 64-slot block per
(tile, direction, copy), block base ``((copy*t_n + tile)*19 + q)*64`` and the
slot inside the block given by the direction's layout function.

B200 addition: ``LayoutKind.ZXY`` (z fastest) and ``LayoutTable.B200``, which
is the reference OPTIMIZED table with the four XY diagonals (NE, NW, SE, SW)
switched to ZXY.  With it every 32-byte fp64 sector of a block is consumed by
exactly one destination tile in the pull gather (304
sectors per tile = the 2*19*8 B/node minimum, vs 344 for OPTIMIZED), so the
step's DRAM traffic does not depend on L2 reuse between tiles.  It is the
solver's default table for both precisions.

``FieldStore`` keeps the reference API but lives in GPU memory (a torch
tensor); canonical I/O runs the library's scatter/gather kernels.
"""

import enum

import numpy as np
import torch

from . import _native as nat
from .lattice import Q, TILE_X, TILE_Y, TILE_Z, direction_index


class LayoutKind(enum.Enum):
    XYZ = "xyz"
    YXZ = "yxz"
    ZIGZAG_NE = "zigzag_ne"
    ZXY = "zxy"


class LayoutTable(enum.Enum):
    OPTIMIZED = "optimized"
    XYZ = "xyz"
    B200 = "b200"


TABLE_CODE = {LayoutTable.XYZ: nat.TABLE_XYZ, LayoutTable.OPTIMIZED: nat.TABLE_OPTIMIZED,
              LayoutTable.B200: nat.TABLE_B200}


def _in_tile(x, y, z):
    for c in (x, y, z):
        if not 0 <= int(c) <= 3:
            raise ValueError(f"intra-tile coordinate out of range 0..3: {c}")
    return int(x), int(y), int(z)


def l_xyz(x, y, z):
    x, y, z = _in_tile(x, y, z)
    return x + 4 * y + 16 * z


def l_yxz(x, y, z):
    x, y, z = _in_tile(x, y, z)
    return y + 4 * x + 16 * z


def l_zigzag_ne(x, y, z):
    """layout.py:55-58: z-pairs of an (x, y) column in adjacent slots."""
    x, y, z = _in_tile(x, y, z)
    return 2 * (x + 3 * y + ((x + 1) & 4) * (3 - y)) + (z & 1) + 16 * (z & 2)


def l_zxy(x, y, z):
    """z fastest: the 4 z-nodes of an (x, y) column fill one fp64 sector."""
    x, y, z = _in_tile(x, y, z)
    return z + 4 * x + 16 * y


LAYOUT_FUNCTIONS = {LayoutKind.XYZ: l_xyz, LayoutKind.YXZ: l_yxz,
                    LayoutKind.ZIGZAG_NE: l_zigzag_ne, LayoutKind.ZXY: l_zxy}


def offsets(kind):
    fn = LAYOUT_FUNCTIONS[kind]
    return np.array([fn(x, y, z) for x, y, z in zip(TILE_X, TILE_Y, TILE_Z)])


def _assign(groups):
    out = {}
    for kind, names in groups.items():
        for n in names:
            out[direction_index(n)] = kind
    return out


_OPTIMIZED = _assign({
    LayoutKind.XYZ: ("O", "N", "S", "T", "B", "NT", "NB", "ST", "SB"),
    LayoutKind.ZIGZAG_NE: ("NE", "SE"),
    LayoutKind.YXZ: ("E", "W", "ET", "EB", "NW", "SW", "WT", "WB")})
_B200 = _assign({
    LayoutKind.XYZ: ("O", "N", "S", "T", "B", "NT", "NB", "ST", "SB"),
    LayoutKind.ZXY: ("NE", "NW", "SE", "SW"),
    LayoutKind.YXZ: ("E", "W", "ET", "EB", "WT", "WB")})


def layout_for_direction(direction, table=LayoutTable.OPTIMIZED):
    """layout.py:89-96."""
    direction = int(direction)
    if not 0 <= direction < Q:
        raise ValueError(f"direction index out of range 0..18: {direction}")
    if table is LayoutTable.XYZ:
        return LayoutKind.XYZ
    if table is LayoutTable.B200:
        return _B200[direction]
    return _OPTIMIZED[direction]


def default_table(precision):
    """Reference defaults (layout.py:99-105): OPTIMIZED for f64, XYZ for f32.
    The Solver itself defaults to LayoutTable.B200 for both."""
    if precision == "f64":
        return LayoutTable.OPTIMIZED
    if precision == "f32":
        return LayoutTable.XYZ
    raise ValueError(f"unknown precision: {precision!r}")


def table_permutations(table):
    """(19, 64) canonical slot -> block offset (layout.py:108-112)."""
    return np.stack([offsets(layout_for_direction(q, table)) for q in range(Q)])


def value_address(tile_index, direction, copy, x, y, z, *, t_n,
                  table=LayoutTable.OPTIMIZED):
    """Flat index of one value in the two-copy store (layout.py:115-132)."""
    tile_index, direction = int(tile_index), int(direction)
    if not 0 <= tile_index < t_n:
        raise ValueError(f"tile index out of range 0..{t_n - 1}: {tile_index}")
    if not 0 <= direction < Q:
        raise ValueError(f"direction index out of range 0..18: {direction}")
    if int(copy) not in (0, 1):
        raise ValueError(f"copy flag must be 0 or 1: {copy}")
    fn = LAYOUT_FUNCTIONS[layout_for_direction(direction, table)]
    return ((int(copy) * t_n + tile_index) * Q + direction) * 64 + fn(x, y, z)


def _as_device(values, dtype, device):
    if isinstance(values, torch.Tensor):
        return values.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(values)).to(device=device, dtype=dtype)


class FieldStore:
    """Two copies of all f_q in per-tile 64-slot blocks, resident on the GPU
    (layout.py:135-167).  ``flat`` is a torch tensor of 2*t_n*19*64 values."""

    def __init__(self, t_n, table=LayoutTable.OPTIMIZED, dtype=np.float64, device=None,
                 zero=True):
        self.device = nat.require_cuda(device)
        self.t_n = int(t_n)
        self.table = table
        self.dtype = np.dtype(dtype)
        self.code = nat.code_of(self.dtype)
        self.tdtype = nat.torch_dtype(self.code)
        alloc = torch.zeros if zero else torch.empty   # Solver overwrites every slot
        self.flat = alloc(2 * self.t_n * Q * 64, dtype=self.tdtype, device=self.device)
        self.perms = table_permutations(table)

    def copy_tensor(self, copy):
        if int(copy) not in (0, 1):
            raise ValueError(f"copy flag must be 0 or 1: {copy}")
        n = self.t_n * Q * 64
        return self.flat[int(copy) * n:(int(copy) + 1) * n]

    def blocks(self, copy):
        """(t_n, 19, 64) view of one copy (a device tensor)."""
        return self.copy_tensor(copy).view(self.t_n, Q, 64)

    def fill_canonical(self, copy, values):
        """Scatter (19, t_n, 64) canonical values into one copy."""
        nat.require_cuda(self.device)
        src = _as_device(values, self.tdtype, self.device)
        if tuple(src.shape) != (Q, self.t_n, 64):
            raise ValueError(f"expected shape (19, {self.t_n}, 64), got {tuple(src.shape)}")
        nat.call("tlbm_from_canonical", nat.ptr(src), self.code, TABLE_CODE[self.table],
                 self.t_n, nat.ptr(self.copy_tensor(copy)), nat.stream_ptr(self.device))

    def read_canonical(self, copy, device=False):
        """Gather one copy to (19, t_n, 64) canonical order; numpy unless
        ``device=True`` (then the torch tensor stays on the GPU)."""
        nat.require_cuda(self.device)
        out = torch.empty((Q, self.t_n, 64), dtype=self.tdtype, device=self.device)
        nat.call("tlbm_to_canonical", nat.ptr(self.copy_tensor(copy)), self.code,
                 TABLE_CODE[self.table], self.t_n, nat.ptr(out), nat.stream_ptr(self.device))
        return out if device else out.cpu().numpy()


class CompactFieldStore(FieldStore):
    """Two copies holding only the non-solid slots of every block, in the
    canonical XYZ slot order (an extension of the paper's layout;
    csrc/compact.cu).  Tile t's 19 blocks start at ``base[t]`` = 19 x
    (non-solid nodes of the tiles before t), each ``nf[t]`` values long, slot
    j at ``rank[t, j]`` (its index among the tile's non-solid slots, 255 for
    a solid slot).  ``flat`` holds 2 x 19 x n_fn values.

    Canonical I/O goes through the paper's block layout: ``to_blocks`` /
    ``from_blocks`` convert one copy to and from a (t_n, 19, 64) XYZ block
    store, whose solid slots read as the rest state w_q."""

    def __init__(self, tiling, table=LayoutTable.XYZ, dtype=np.float64):
        if table is not LayoutTable.XYZ:
            raise ValueError(f"compact storage keeps blocks in XYZ order; table must be xyz, "
                             f"not {table.value}")
        self.device = nat.require_cuda(tiling.device)
        self.t_n = int(tiling.t_n)
        self.n_fn = int(tiling.n_fn)
        self.table = table
        self.dtype = np.dtype(dtype)
        self.code = nat.code_of(self.dtype)
        self.tdtype = nat.torch_dtype(self.code)
        self.perms = table_permutations(table)
        self.nf = tiling.counts
        base = torch.zeros(max(self.t_n, 1), dtype=torch.int64, device=self.device)
        if self.t_n > 1:
            base[1:self.t_n] = torch.cumsum(self.nf[:-1].to(torch.int64), 0) * Q
        self.base = base[:self.t_n]
        self.rank = torch.empty((max(self.t_n, 1), 64), dtype=torch.uint8,
                                device=self.device)[:self.t_n]
        nat.call("tlbm_compact_ranks", nat.ptr(tiling.meta), self.t_n, nat.ptr(self.rank),
                 nat.stream_ptr(self.device))
        self.flat = torch.empty(2 * Q * self.n_fn, dtype=self.tdtype, device=self.device)

    def node_records(self, tiling):
        """Per-node records for the node-parallel step (tlbm_compact_nodes):
        ``node_meta`` (n_fn,) int32, ``node_rec`` (n_fn, 4) int32, ``unit_tile``
        (ceil(n_fn / 64),) int32 and ``entries`` (t_n, 27, 2) int32 -- 20 B
        per node + 216 B per tile; built once and cached."""
        if getattr(self, "_nodes", None) is None:
            dev = self.device
            n = max(self.n_fn, 1)
            rec = {"node_meta": torch.empty(n, dtype=torch.int32, device=dev),
                   "node_rec": torch.empty((n, 4), dtype=torch.int32, device=dev),
                   "unit_tile": torch.empty((n + 63) // 64, dtype=torch.int32, device=dev),
                   "entries": torch.empty((max(self.t_n, 1), 27, 2), dtype=torch.int32,
                                          device=dev)}
            nat.call("tlbm_compact_nodes", nat.ptr(tiling.meta), nat.ptr(tiling.nbr), self.t_n,
                     self.n_fn, nat.ptr(self.base), nat.ptr(self.nf), nat.ptr(self.rank),
                     nat.ptr(rec["node_meta"]), nat.ptr(rec["node_rec"]),
                     nat.ptr(rec["unit_tile"]), nat.ptr(rec["entries"]),
                     nat.stream_ptr(dev))
            self._nodes = rec
        return self._nodes

    def node_range(self, tile_begin, tile_end):
        """Store-order node range [n0, n1) of tiles [tile_begin, tile_end)."""
        if getattr(self, "_node_prefix", None) is None:
            self._node_prefix = np.concatenate(
                [(self.base // Q).cpu().numpy(), [self.n_fn]]).astype(np.int64)
        return int(self._node_prefix[tile_begin]), int(self._node_prefix[tile_end])

    def copy_tensor(self, copy):
        if int(copy) not in (0, 1):
            raise ValueError(f"copy flag must be 0 or 1: {copy}")
        n = Q * self.n_fn
        return self.flat[int(copy) * n:(int(copy) + 1) * n]

    def _convert(self, src, dst, to_compact):
        nat.call("tlbm_compact_convert", nat.ptr(src), nat.ptr(dst), self.code,
                 TABLE_CODE[self.table], self.t_n, nat.ptr(self.base), nat.ptr(self.nf),
                 nat.ptr(self.rank), int(to_compact), nat.stream_ptr(self.device))

    def to_blocks(self, copy):
        """One copy expanded to the paper's (t_n*19*64,) block store (a new
        tensor; solid slots hold the rest state w_q)."""
        out = torch.empty(self.t_n * Q * 64, dtype=self.tdtype, device=self.device)
        self._convert(self.copy_tensor(copy), out, False)
        return out

    def from_blocks(self, copy, blocks):
        self._convert(blocks, self.copy_tensor(copy), True)

    def blocks(self, copy):
        """(t_n, 19, 64) blocks of one copy (an expanded copy, not a view)."""
        return self.to_blocks(copy).view(self.t_n, Q, 64)

    def fill_canonical(self, copy, values):
        nat.require_cuda(self.device)
        src = _as_device(values, self.tdtype, self.device)
        if tuple(src.shape) != (Q, self.t_n, 64):
            raise ValueError(f"expected shape (19, {self.t_n}, 64), got {tuple(src.shape)}")
        tmp = torch.empty(self.t_n * Q * 64, dtype=self.tdtype, device=self.device)
        nat.call("tlbm_from_canonical", nat.ptr(src), self.code, TABLE_CODE[self.table],
                 self.t_n, nat.ptr(tmp), nat.stream_ptr(self.device))
        self.from_blocks(copy, tmp)

    def read_canonical(self, copy, device=False):
        nat.require_cuda(self.device)
        tmp = self.to_blocks(copy)
        out = torch.empty((Q, self.t_n, 64), dtype=self.tdtype, device=self.device)
        nat.call("tlbm_to_canonical", nat.ptr(tmp), self.code, TABLE_CODE[self.table],
                 self.t_n, nat.ptr(out), nat.stream_ptr(self.device))
        return out if device else out.cpu().numpy()

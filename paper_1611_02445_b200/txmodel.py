"""Bandwidth model of the step (txmodel.py:48-68) used by the bench's roofline.

B_node = 2 * q * n_d bytes moved per non-solid node per step (each value read
once and written once): 304 B fp64, 152 B fp32.  The
per-tile metadata the B200 kernel also reads (64 x 4 B node words + 27 x 4 B
neighbour row per tile) is reported separately by ``metadata_bytes``.
"""

SEGMENT_BYTES = 32
_PRECISION_BYTES = {"f64": 8, "f32": 4}


def value_bytes(precision):
    if precision not in _PRECISION_BYTES:
        raise ValueError(f"unknown precision: {precision!r}")
    return _PRECISION_BYTES[precision]


def m_node(q=19, n_d=8):
    if q <= 0 or n_d <= 0:
        raise ValueError(f"q and n_d must be positive: q={q}, n_d={n_d}")
    return q * n_d


def b_node(q=19, n_d=8):
    return 2 * m_node(q, n_d)


def flop_per_byte(flop_count, bytes_per_node):
    if bytes_per_node <= 0:
        raise ValueError(f"bytes per node must be positive: {bytes_per_node}")
    if flop_count < 0:
        raise ValueError(f"FLOP count must be non-negative: {flop_count}")
    return flop_count / bytes_per_node


class PerfModel:
    """Bandwidth-bound cost model (txmodel.py:32-45): per-node byte minima."""

    def __init__(self, q=19, n_d=8, n_t=1, segment_bytes=SEGMENT_BYTES):
        self.q, self.n_d, self.n_t, self.segment_bytes = q, n_d, n_t, segment_bytes

    def __repr__(self):
        return (f"PerfModel(q={self.q}, n_d={self.n_d}, n_t={self.n_t}, "
                f"segment_bytes={self.segment_bytes})")

    def __eq__(self, other):
        return isinstance(other, PerfModel) and vars(self) == vars(other)

    def m_node(self):
        return m_node(self.q, self.n_d)

    def b_node(self):
        return b_node(self.q, self.n_d)


def metadata_bytes(t_n):
    """Bytes of per-tile metadata one step reads: node words + neighbour row."""
    return t_n * (64 * 4 + 27 * 4)


# -- 32-byte segment model of the gather (txmodel.py:71-252) -------------------
# Host analytics: replays, per warp of a tile (z-pairs, lattice.py:97-106),
# which aligned 32-byte segments of which source tile each direction's pull
# touches, for a layout table.  ncu's dram/lts sector counts are the measured
# counterpart (profiles/).

from dataclasses import dataclass as _dataclass

import numpy as _np

from . import lattice as _lat
from . import layout as _lay
from .lattice import TILE_X, TILE_Y, TILE_Z  # noqa: F401,E402 (reference namespace)


@_dataclass
class TransactionReport:
    precision: str
    table: object
    per_direction_reads: dict
    tile_read_total: int
    tile_read_min: int
    read_overhead: float
    t_n: int = None
    write_segments_min: int = None
    write_segments_model: int = None
    nodetype_read_segments: int = None
    read_segments_min: int = None
    read_segments_model: int = None
    total_min: int = None
    total_model: int = None
    tilemap_values_read: int = None
    overhead_vs_min: float = None
    nodetype_bytes_convention: int = 2


def _gather_plan(q, kind, n_d):
    """Per destination slot j: (warp, source-tile delta, segment, source slot)."""
    per_seg = SEGMENT_BYTES // n_d
    e = _lat.E_VECTORS[q]
    fn = _lay.LAYOUT_FUNCTIONS[kind]
    plan = []
    for j in range(64):
        s = (_lat.TILE_X[j] - e[0], _lat.TILE_Y[j] - e[1], _lat.TILE_Z[j] - e[2])
        delta = tuple(-1 if c < 0 else (1 if c > 3 else 0) for c in s)
        lx, ly, lz = (int(c) & 3 for c in s)
        plan.append((j, int(_lat.TILE_Z[j]) >> 1, delta, fn(lx, ly, lz) // per_seg,
                     lx + 4 * ly + 16 * lz))
    return plan


def count_direction_reads(direction, kind, precision):
    """Distinct (warp, source tile, segment) triples of one direction's pull
    over a fully fluid tile (txmodel.py:112-121)."""
    plan = _gather_plan(int(direction), kind, value_bytes(precision))
    return len({(w, d, s) for _, w, d, s, _ in plan})


def count_tile_overheads(table, precision):
    """Per-direction and per-tile read segments of a layout table
    (txmodel.py:124-142); B200 table: 320 f64 (304 under the whole-tile model)."""
    n_d = value_bytes(precision)
    per = {_lat.direction_name(q): count_direction_reads(q, _lay.layout_for_direction(q, table),
                                                         precision) for q in range(19)}
    total = sum(per.values())
    minimum = 19 * (64 * n_d // SEGMENT_BYTES)
    return TransactionReport(precision, table, per, total, minimum, total / minimum - 1.0)


def count_tile_reads_whole_tile(table, precision):
    """Segments per tile when the whole tile is the request unit (L1 dedupes
    the two warps on B200): distinct (source tile, segment) pairs."""
    n_d = value_bytes(precision)
    total = 0
    for q in range(19):
        plan = _gather_plan(q, _lay.layout_for_direction(q, table), n_d)
        total += len({(d, s) for _, _, d, s, _ in plan})
    return total


def geometry_transaction_totals(grid, geometry, table, precision):
    """The segment model over a concrete tiling with solid skips
    (txmodel.py:176-252)."""
    import itertools

    if grid.a != 4:
        raise ValueError("transaction model is defined for 4^3-node tiles")
    n_d = value_bytes(precision)
    segs_per_block = 64 * n_d // SEGMENT_BYTES
    t_n = grid.t_n
    rep = count_tile_overheads(table, precision)
    nx, ny, nz = geometry.shape
    px, py, pz = grid.padded_dims
    ns = _np.zeros((px, py, pz), dtype=bool)
    ns[:nx, :ny, :nz] = geometry.types != 0
    ne = grid.non_empty
    dest = ns[ne[:, 0:1] + _lat.TILE_X, ne[:, 1:2] + _lat.TILE_Y, ne[:, 2:3] + _lat.TILE_Z]
    deltas = list(itertools.product((-1, 0, 1), repeat=3))
    mesh = _np.array(grid.tile_map.shape)
    coords = ne.astype(_np.int64) // 4
    nbr = _np.full((t_n, 27), -1, dtype=_np.int64)
    for k, d in enumerate(deltas):
        c = coords + _np.asarray(d)
        ok = _np.all((c >= 0) & (c < mesh), axis=1)
        nbr[ok, k] = grid.tile_map[c[ok, 0], c[ok, 1], c[ok, 2]]
    reads = 0
    for q in range(19):
        groups = {}
        for j, w, d, s, src in _gather_plan(q, _lay.layout_for_direction(q, table), n_d):
            groups.setdefault((w, d, s), []).append((j, src))
        for (w, d, s), members in groups.items():
            nb = nbr[:, deltas.index(d)]
            ok = nb >= 0
            dst = _np.array([m[0] for m in members])
            src = _np.array([m[1] for m in members])
            src_ns = dest[_np.where(ok, nb, 0)[:, None], src[None, :]]
            reads += int(_np.count_nonzero((dest[:, dst] & src_ns).any(axis=1) & ok))
    writes = 0
    perms = _lay.table_permutations(table)
    for q in range(19):
        seg = perms[q] // (SEGMENT_BYTES // n_d)
        for k in range(segs_per_block):
            writes += int(_np.count_nonzero(dest[:, _np.flatnonzero(seg == k)].any(axis=1)))
    write_min = t_n * 19 * segs_per_block
    nodetype = t_n * (64 * 2 // SEGMENT_BYTES)
    rep.t_n = t_n
    rep.write_segments_min = write_min
    rep.write_segments_model = writes
    rep.nodetype_read_segments = nodetype
    rep.read_segments_min = write_min + nodetype
    rep.read_segments_model = reads + nodetype
    rep.total_min = 2 * write_min + nodetype
    rep.total_model = writes + reads + nodetype
    rep.tilemap_values_read = 27 * t_n
    rep.overhead_vs_min = rep.total_model / rep.total_min - 1.0
    return rep

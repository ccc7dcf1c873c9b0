"""D3Q19 velocity set, weights and the intra-tile slot convention.

Mirrors ``tilelbm.lattice`` (reference ``lattice.py:22-120``): same direction
order (O, E, N, W, S, T, B, NE, NW, SE, SW, NT, NB, ST, SB, ET, EB, WT, WB),
same weights 1/3, 1/18, 1/36 and the same slot numbering
``j = x + 4*y + 16*z`` inside a 4^3 tile.  The CUDA kernels bake the identical
tables in as compile-time constants (``csrc/d3q19.cuh``); a CPU test checks
both agree.
"""

from fractions import Fraction

import numpy as np

Q = 19
TILE = 4
SLOTS = TILE ** 3

DIRECTION_NAMES = ("O", "E", "N", "W", "S", "T", "B",
                   "NE", "NW", "SE", "SW", "NT", "NB", "ST", "SB",
                   "ET", "EB", "WT", "WB")

_UNIT = {"E": (1, 0, 0), "W": (-1, 0, 0), "N": (0, 1, 0), "S": (0, -1, 0),
         "T": (0, 0, 1), "B": (0, 0, -1)}


def _vector_of(name):
    if name == "O":
        return (0, 0, 0)
    if len(name) == 1:
        return _UNIT[name]
    a, b = _UNIT[name[0]], _UNIT[name[1]]
    return tuple(i + j for i, j in zip(a, b))


E_VECTORS = np.array([_vector_of(n) for n in DIRECTION_NAMES], dtype=np.int64)
INDEX_BY_NAME = {n: i for i, n in enumerate(DIRECTION_NAMES)}

WEIGHTS_EXACT = tuple(Fraction(1, 3) if q == 0 else
                      Fraction(1, 18) if q < 7 else Fraction(1, 36)
                      for q in range(Q))
WEIGHTS = np.array([float(w) for w in WEIGHTS_EXACT])

CS2 = 1.0 / 3.0
DELTA_X = 1.0
DELTA_T = 1.0

OPPOSITE = np.array([int(np.flatnonzero((E_VECTORS == -E_VECTORS[q]).all(1))[0])
                     for q in range(Q)], dtype=np.int64)

AXIS_DIRECTIONS = tuple(range(1, 7))
DIAGONAL_DIRECTIONS = tuple(range(7, 19))


def _q(i):
    i = int(i)
    if i < 0 or i >= Q:
        raise ValueError(f"direction index out of range 0..18: {i}")
    return i


def direction_vector(i):
    return tuple(int(c) for c in E_VECTORS[_q(i)])


def direction_name(i):
    return DIRECTION_NAMES[_q(i)]


def direction_index(name):
    if name not in INDEX_BY_NAME:
        raise ValueError(f"unknown direction name: {name!r}")
    return INDEX_BY_NAME[name]


def weight(i):
    return WEIGHTS_EXACT[_q(i)]


def opposite(i):
    return int(OPPOSITE[_q(i)])


def thread_linear_index(tx, ty, tz):
    """Slot of intra-tile node (tx, ty, tz): tx + 4 ty + 16 tz (lattice.py:97-106)."""
    c = [int(v) for v in (tx, ty, tz)]
    if any(v < 0 or v >= TILE for v in c):
        raise ValueError(f"intra-tile coordinate out of range 0..3: {tuple(c)}")
    return c[0] + TILE * c[1] + TILE * TILE * c[2]


def node_coords(j):
    """Inverse of ``thread_linear_index`` (lattice.py:109-114)."""
    j = int(j)
    if j < 0 or j >= SLOTS:
        raise ValueError(f"tile slot out of range 0..63: {j}")
    return j & 3, (j >> 2) & 3, j >> 4


_SLOT = np.arange(SLOTS)
TILE_X = _SLOT & 3
TILE_Y = (_SLOT >> 2) & 3
TILE_Z = (_SLOT >> 4) & 3

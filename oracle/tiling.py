"""Tiling, neighbour map and layout tables restated in numpy (oracle side).

build_tiling      tiling.py:51-83   pad with SOLID, any-non-solid per 4^3 tile,
                                    compact in (z outer, y, x inner) scan order
neighbor_indices  txmodel.py:145-160  tile index per delta, -1 absent/outside
                                    (optional periodic wrap -- extension)
nonsolid_blocks   txmodel.py:163-173  (t_n, 64) canonical non-solid flags
layout tables     layout.py:45-112    per-direction slot permutations
"""

import itertools

import numpy as np

DELTAS27 = tuple(itertools.product((-1, 0, 1), repeat=3))
SLOT = np.arange(64)
SX, SY, SZ = SLOT & 3, (SLOT >> 2) & 3, SLOT >> 4


def build_tiling(types, a=4):
    nx, ny, nz = types.shape
    ntx, nty, ntz = (-(-n // a) for n in (nx, ny, nz))
    occ = np.zeros((ntx * a, nty * a, ntz * a), dtype=bool)
    occ[:nx, :ny, :nz] = types != 0
    occ = occ.reshape(ntx, a, nty, a, ntz, a).any(axis=(1, 3, 5))
    order = np.flatnonzero(occ.transpose(2, 1, 0).ravel())
    tz, ty, tx = np.unravel_index(order, (ntz, nty, ntx))
    tile_map = np.full((ntx, nty, ntz), -1, dtype=np.int32)
    tile_map[tx, ty, tz] = np.arange(order.size, dtype=np.int32)
    non_empty = (np.stack([tx, ty, tz], axis=1) * a).astype(np.int32)
    return tile_map, non_empty


def neighbor_indices(tile_map, non_empty, deltas=DELTAS27, periodic=(False,) * 3,
                     a=4):
    mesh = np.array(tile_map.shape)
    coords = non_empty.astype(np.int64) // a
    out = np.full((len(non_empty), len(deltas)), -1, dtype=np.int64)
    for k, d in enumerate(deltas):
        nb = coords + np.asarray(d, dtype=np.int64)
        for ax in range(3):
            if periodic[ax]:
                nb[:, ax] %= mesh[ax]
        ok = np.all((nb >= 0) & (nb < mesh), axis=1)
        out[ok, k] = tile_map[nb[ok, 0], nb[ok, 1], nb[ok, 2]]
    return out


def nonsolid_blocks(types, non_empty, a=4):
    nx, ny, nz = types.shape
    pdims = [(-(-n // a)) * a for n in (nx, ny, nz)]
    ns = np.zeros(pdims, dtype=bool)
    ns[:nx, :ny, :nz] = types != 0
    return ns[non_empty[:, 0:1] + SX, non_empty[:, 1:2] + SY,
              non_empty[:, 2:3] + SZ]


def tile_types(types, non_empty, a=4):
    """(t_n, 64) canonical node tags of every tile, padding = SOLID (0)."""
    nx, ny, nz = types.shape
    pdims = [(-(-n // a)) * a for n in (nx, ny, nz)]
    t = np.zeros(pdims, dtype=np.uint8)
    t[:nx, :ny, :nz] = types
    return t[non_empty[:, 0:1] + SX, non_empty[:, 1:2] + SY,
             non_empty[:, 2:3] + SZ]


# -- layouts (layout.py:45-112) plus the z-fastest kind used by the B200
#    table -------------------------------------------------

LAYOUT_FUNCS = {
    "xyz": lambda x, y, z: x + 4 * y + 16 * z,
    "yxz": lambda x, y, z: y + 4 * x + 16 * z,
    "zigzag_ne": lambda x, y, z: 2 * (x + 3 * y + ((x + 1) & 4) * (3 - y))
    + (z & 1) + 16 * (z & 2),
    "zxy": lambda x, y, z: z + 4 * x + 16 * y,
}

_NAMES = ("O", "E", "N", "W", "S", "T", "B", "NE", "NW", "SE", "SW",
          "NT", "NB", "ST", "SB", "ET", "EB", "WT", "WB")


def _table(spec):
    kinds = []
    for name in _NAMES:
        for kind, names in spec.items():
            if name in names:
                kinds.append(kind)
                break
    return tuple(kinds)


TABLES = {
    "xyz": ("xyz",) * 19,
    "optimized": _table({"xyz": ("O", "N", "S", "T", "B", "NT", "NB", "ST", "SB"),
                         "zigzag_ne": ("NE", "SE"),
                         "yxz": ("E", "W", "ET", "EB", "NW", "SW", "WT", "WB")}),
    "b200": _table({"xyz": ("O", "N", "S", "T", "B", "NT", "NB", "ST", "SB"),
                    "zxy": ("NE", "NW", "SE", "SW"),
                    "yxz": ("E", "W", "ET", "EB", "WT", "WB")}),
}


def table_permutations(table):
    kinds = TABLES[getattr(table, "value", table)]
    return np.stack([np.array([LAYOUT_FUNCS[k](x, y, z)
                               for x, y, z in zip(SX, SY, SZ)]) for k in kinds])


def to_blocks(canonical, table):
    """(19, t_n, 64) canonical -> (t_n, 19, 64) stored blocks (layout.py:155-159)."""
    perms = table_permutations(table)
    t_n = canonical.shape[1]
    out = np.zeros((t_n, 19, 64), dtype=canonical.dtype)
    for q in range(19):
        out[:, q, perms[q]] = canonical[q]
    return out


def from_blocks(blocks, table):
    """(t_n, 19, 64) stored blocks -> (19, t_n, 64) canonical (layout.py:161-167)."""
    perms = table_permutations(table)
    return np.stack([blocks[:, q, perms[q]] for q in range(19)])


def meta_words(types, non_empty, periodic=(False,) * 3, a=4):
    """(t_n, 64) u32 per-slot node words the device tiler must produce,
    restated from the step contract:
      bit 0       slot is a non-solid node inside the domain (R1)
      bit q 1..18 the pull source n - e_q is inside the domain (wrapped on a
                  periodic axis) and non-solid, i.e. g_q is a neighbour value
                  and not the halfway bounce-back fill (R2)
      bits 19-21  the node tag (geometry.py:17-24)
      bits 22-24  the Zou-He face 2*axis + (0 low | 1 high) of an inlet /
                  outlet node (classify_boundary_faces, boundaries.py:95-129)
    """
    from .dense import face_ids
    from .numerics import E
    nx, ny, nz = types.shape
    dims = np.array([nx, ny, nz])
    x = non_empty[:, 0:1].astype(np.int64) + SX
    y = non_empty[:, 1:2].astype(np.int64) + SY
    z = non_empty[:, 2:3].astype(np.int64) + SZ
    inside = (x < nx) & (y < ny) & (z < nz)
    xc, yc, zc = np.minimum(x, nx - 1), np.minimum(y, ny - 1), np.minimum(z, nz - 1)
    tag = np.where(inside, types[xc, yc, zc], 0).astype(np.uint32)
    w = np.where(tag != 0, 1 | (tag << 19), 0).astype(np.uint32)
    for q in range(1, 19):
        s = [x - E[q][0], y - E[q][1], z - E[q][2]]
        ok = np.ones(x.shape, dtype=bool)
        for ax in range(3):
            if periodic[ax]:
                s[ax] = s[ax] % dims[ax]
            ok &= (s[ax] >= 0) & (s[ax] < dims[ax])
        sx, sy, sz = (np.clip(s[ax], 0, dims[ax] - 1) for ax in range(3))
        link = ok & (types[sx, sy, sz] != 0) & (tag != 0)
        w |= np.where(link, np.uint32(1 << q), np.uint32(0))
    f = face_ids(types, periodic)
    face = np.where(inside, f[xc, yc, zc], -1)
    io = (tag == 3) | (tag == 4)
    w |= np.where(io, face.astype(np.int64) << 22, 0).astype(np.uint32)
    return w

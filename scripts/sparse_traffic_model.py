"""DRAM-granule model of one step on a sparse geometry (analysis tool).

For every fluid (non-solid) node and direction, the value the pull gather
reads (neighbour slot, or the node's own opposite slot under halfway
bounce-back) and the value it writes, as element addresses of the field
store -- either the paper's layout (`[tile][q][64]`, `layout.py:115-132`) or
a compacted variant that keeps only the non-solid slots of every block, in
layout order.  Prints the unique 32/64/128-byte granules read and written
per step, per fluid node, to compare with ncu's dram__bytes_read/write
(profiles/r1b_ncu_sparse_dram.json).

    python scripts/sparse_traffic_model.py --porosity 0.2 [--n 256] [--table b200]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import tiling as ot  # noqa: E402
from paper_1611_02445_b200 import layout, workloads  # noqa: E402
from paper_1611_02445_b200.lattice import E_VECTORS, OPPOSITE  # noqa: E402


def model(types, table, n_d, compact, granules=(32, 64, 128)):
    tile_map, non_empty = ot.build_tiling(types)
    t_n = len(non_empty)
    ns = ot.nonsolid_blocks(types, non_empty)                    # (t_n, 64) canonical
    perm = np.asarray(layout.table_permutations(table))           # (19, 64) slot of canonical j
    nf = ns.sum(axis=1)
    if compact:
        # rank of canonical slot j among the non-solid slots of its block, in
        # the layout order of direction q
        rank = np.zeros((19, t_n, 64), dtype=np.int64)
        for q in range(19):
            inv = np.argsort(perm[q])                             # layout position -> canonical
            m = ns[:, inv]                                        # mask in layout order
            r = np.cumsum(m, axis=1) - 1
            rank[q][:, inv] = r
        base = np.concatenate([[0], np.cumsum(19 * nf)[:-1]])

        def addr(t, q, j):
            return base[t] + q * nf[t] + rank[q, t, j]
    else:
        def addr(t, q, j):
            return (t * 19 + q) * 64 + perm[q, j]
    nx, ny, nz = types.shape
    tt, jj = np.nonzero(ns)                                       # fluid (tile, slot)
    x = non_empty[tt, 0] + (jj & 3)
    y = non_empty[tt, 1] + ((jj >> 2) & 3)
    z = non_empty[tt, 2] + (jj >> 4)
    reads, writes = [], []
    for q in range(19):
        e = E_VECTORS[q]
        sx, sy, sz = x - e[0], y - e[1], z - e[2]
        inside = (sx >= 0) & (sx < nx) & (sy >= 0) & (sy < ny) & (sz >= 0) & (sz < nz)
        link = np.zeros_like(inside)
        link[inside] = types[sx[inside], sy[inside], sz[inside]] != 0
        st = np.where(link, tile_map[np.clip(sx, 0, nx - 1) // 4, np.clip(sy, 0, ny - 1) // 4,
                                     np.clip(sz, 0, nz - 1) // 4], tt)
        sj = np.where(link, (sx & 3) + 4 * (sy & 3) + 16 * (sz & 3), jj)
        sq = np.where(link, q, OPPOSITE[q])
        reads.append(addr(st, sq, sj))
        writes.append(addr(tt, np.full_like(tt, q), jj))
    reads, writes = np.concatenate(reads), np.concatenate(writes)
    n_fn = len(tt)
    out = {"t_n": t_n, "n_fn": int(n_fn), "eta_t": float(n_fn / (64 * t_n)),
           "compact": compact, "n_d": n_d}
    for g in granules:
        per = g // n_d
        out[f"read_B_per_node_{g}"] = len(np.unique(reads // per)) * g / n_fn
        out[f"write_B_per_node_{g}"] = len(np.unique(writes // per)) * g / n_fn
        # partially written granules (a DRAM write of them needs the rest)
        w = np.bincount(writes // per)
        out[f"partial_write_granules_per_node_{g}"] = float(((w > 0) & (w < per)).sum() / n_fn)
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--porosity", type=float, default=0.2)
    p.add_argument("--n", type=int, default=256)
    p.add_argument("--table", default="b200")
    p.add_argument("--precision", default="f64")
    a = p.parse_args()
    geo = workloads.sphere_pack(a.porosity, n=a.n)
    n_d = 8 if a.precision == "f64" else 4
    table = layout.LayoutTable(a.table) if a.table in [t.value for t in layout.LayoutTable] \
        else layout.LayoutTable[a.table.upper()]
    for compact in (False, True):
        r = model(geo.types, table, n_d, compact)
        r.update({"porosity": a.porosity, "n": a.n, "table": str(a.table),
                  "precision": a.precision})
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()

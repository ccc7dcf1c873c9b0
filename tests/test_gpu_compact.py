"""GPU: compact tile storage (SimulationConfig(storage="compact"),
csrc/compact.cu, csrc/step_compact.cuh).  The compact store keeps only the
non-solid slots of every block; the arithmetic is the block-store kernel's,
so every result is bit-identical to the paper's layout and to the oracle."""

import numpy as np
import pytest
import torch

from helpers import random_geometry
from oracle import dense, numerics as nm
from paper_1611_02445_b200 import _native as nat
from paper_1611_02445_b200 import geometry, layout, slabs, solver
from test_gpu_step import DTYPES, MODELS, compare, oracle_run, perturbed_eq

pytestmark = pytest.mark.gpu
def make(geo, m=MODELS["inc"], dt=np.float64, table=None, f0=None, storage="compact",
         traversal="tile", **kw):
    cfg = solver.SimulationConfig(fluid=m, tau=0.6, u_max_guard=0.0, table=table,
                                  precision="f64" if dt == np.float64 else "f32",
                                  storage=storage, **kw)
    s = solver.Solver(geo, cfg, traversal=traversal)
    if f0 is not None:
        s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
    return s


def test_store_size_and_canonical_roundtrip():
    geo = geometry.generate_sphere_pack(24, 6, 0.4, seed=3, inlet_velocity=(0, 0, 0.01))
    s = make(geo)
    assert s.store.flat.numel() == 2 * 19 * s.n_fn < 2 * 19 * 64 * s.t_n
    vals = np.random.default_rng(0).random((19, s.t_n, 64))
    s.set_fields_canonical(vals)
    got = s.fields_canonical()
    mask = s.nonsolid_mask()
    assert np.array_equal(got[:, mask], vals[:, mask])
    assert np.array_equal(got[:, ~mask], np.broadcast_to(nm.W[:, None], (19, (~mask).sum())))


def test_rejects_unsupported_configs():
    assert solver.SimulationConfig(storage="compact").table is layout.LayoutTable.XYZ
    for t in ("optimized", "b200"):
        with pytest.raises(ValueError):
            solver.SimulationConfig(storage="compact", table=t)
    with pytest.raises(ValueError):
        solver.SimulationConfig(storage="sparse")


@pytest.mark.parametrize("traversal", ["tile", "nodes"])
@pytest.mark.parametrize("dn", DTYPES)
def test_cavity64_1000_steps_compact(c_oracle, dn, traversal):
    dt = DTYPES[dn]
    geo = geometry.generate_cavity3d(64)
    m = MODELS["inc"]
    s = make(geo, m, dt, traversal=traversal)
    assert (s.nodes is not None) == (traversal == "nodes")
    s.run(1000)
    compare(s, oracle_run(c_oracle, geo, m, dt, dense.init_equilibrium(geo.shape, m, dt), 1000),
            dt)


@pytest.mark.parametrize("traversal", ["tile", "nodes"])
@pytest.mark.parametrize("seed", range(6))
def test_random_geometries_compact(c_oracle, seed, traversal):
    """Mixed solid / fluid / bounce-back / inlet / outlet geometries, both
    dtypes and fluid models: bit-exact vs the oracle."""
    rng = np.random.default_rng(1300 + seed)
    shape = tuple(int(v) for v in rng.integers(5, 26, size=3))
    t = random_geometry(rng, shape)
    geo = geometry.Geometry(t, inlet_velocity=(0.0, 0.01, 0.02), outlet_density=1.0)
    for dt in (np.float64, np.float32):
        for m in MODELS.values():
            f0 = perturbed_eq(shape, m, dt, (0.0, 0.0, 0.01), seed)
            want = oracle_run(c_oracle, geo, m, dt, f0, 15)
            s = make(geo, m, dt, None, f0, traversal=traversal)
            s.step(15)
            compare(s, want, dt)


@pytest.mark.parametrize("kw", [{}, {"collision": "mrt"}, {"arithmetic": "fma"},
                                {"collision": "mrt", "arithmetic": "fma"},
                                {"fluid": "quasi-compressible", "precision": "f32"}])
def test_compact_equals_blocks(kw):
    """Same configuration, both storages, 70 steps (graph replay for the
    compact one): identical canonical fields and macroscopic readout."""
    geo = geometry.generate_sphere_pack(32, 8, 0.45, seed=6, inlet_velocity=(0, 0, 0.02))
    runs = []
    for storage, trav in (("blocks", "tile"), ("compact", "tile"), ("compact", "nodes")):
        cfg = solver.SimulationConfig(tau=0.6, u_max_guard=0.0, storage=storage,
                                      **({"fluid": "incompressible"} | kw))
        s = solver.Solver(geo, cfg, traversal=trav)
        s.init_equilibrium(1.0, (0.0, 0.0, 0.01))
        s.step(70, graph=(storage == "compact"))
        mask = s.nonsolid_mask(device=True)
        rho, u, _ = s.macroscopic(device=True)
        runs.append((s.fields_canonical(device=True)[:, mask], rho[mask], u[:, mask]))
    for other in runs[1:]:
        for a, b in zip(runs[0], other):
            assert torch.equal(a, b)


@pytest.mark.parametrize("variant", [nat.PROPAGATION_ONLY, nat.READ_WRITE_ONLY])
def test_ladder_variants_compact(variant):
    geo = geometry.generate_sphere_pack(24, 6, 0.5, seed=2, inlet_velocity=(0, 0, 0.01))
    f0 = perturbed_eq(geo.shape, MODELS["inc"], np.float64, seed=5)
    runs = []
    for storage, trav in (("blocks", "tile"), ("compact", "tile"), ("compact", "nodes")):
        s = make(geo, f0=f0, storage=storage, traversal=trav)
        s.step(3, variant=variant)
        runs.append(s.fields_canonical(device=True)[:, s.nonsolid_mask(device=True)])
    assert torch.equal(runs[0], runs[1]) and torch.equal(runs[0], runs[2])


def test_checkpoint_across_storages(tmp_path):
    geo = geometry.generate_sphere_pack(24, 6, 0.5, seed=8, inlet_velocity=(0, 0, 0.02))
    a = make(geo)
    a.step(9)
    a.save_checkpoint(tmp_path / "ck.npz")
    a.step(11)
    b = solver.Solver(geo, solver.SimulationConfig(u_max_guard=0.0, tau=0.6))
    b.load_checkpoint(tmp_path / "ck.npz")
    b.step(11)
    m = b.nonsolid_mask(device=True)
    assert torch.equal(a.fields_canonical(device=True)[:, m], b.fields_canonical(device=True)[:, m])


def test_auto_storage_picks_by_tile_utilisation():
    sparse = geometry.generate_sphere_pack(32, 8, 0.3, seed=1, inlet_velocity=(0, 0, 0.01))
    dense = geometry.generate_channel("square", 16, axis=2, length=16, ends="periodic")
    cfg = solver.SimulationConfig(storage="auto", u_max_guard=0.0)
    s = solver.Solver(sparse, cfg)
    assert s.config.storage == "compact" and s.nodes is not None     # node-parallel step
    assert solver.Solver(dense, cfg).config.storage == "blocks"
    # fp32: compact below eta_t 0.80 only
    eta = sparse_eta = s.n_fn / (64 * s.t_n)
    want = "compact" if eta < solver.AUTO_COMPACT_ETA["f32"] else "blocks"
    cfg32 = solver.SimulationConfig(storage="auto", u_max_guard=0.0, precision="f32")
    assert solver.Solver(sparse, cfg32).config.storage == want, sparse_eta
    assert solver.Solver(sparse, cfg, traversal="tile").nodes is None


def test_node_records_decode():
    """tlbm_compact_nodes records (include/tlbm.h) decoded on the host agree
    with the store's base / count / ranks and the neighbour map: node n of
    tile t at rank r is n = base[t] / 19 + r, its word is the tile's node
    word | slot << 25, and its 18 source ranks are the ranks of the pulled
    slots in their source tiles."""
    from paper_1611_02445_b200 import lattice
    geo = geometry.generate_sphere_pack(24, 6, 0.35, seed=4, inlet_velocity=(0, 0, 0.01))
    s = make(geo, traversal="nodes")
    rec = {k: v.cpu().numpy() for k, v in s.nodes.items()}
    base = s.store.base.cpu().numpy() // 19
    nf = s.store.nf.cpu().numpy()
    rank = s.store.rank.cpu().numpy()
    meta = s.tiling.meta.cpu().numpy().view(np.uint32).reshape(-1)
    nbr = s.tiling.nbr.cpu().numpy()
    ent = rec["entries"].view(np.uint32)
    nm_ = rec["node_meta"].view(np.uint32)
    nr = rec["node_rec"].view(np.uint32)
    e = np.asarray(lattice.E_VECTORS)
    checked = 0
    for t in range(0, s.t_n, max(1, s.t_n // 60)):
        for k in range(27):
            nb = nbr[t, k]
            tt = nb if nb >= 0 else t
            assert ent[t, k, 0] == (base[tt] * 19) & 0xffffffff and ent[t, k, 1] == nf[tt]
        for j in range(64):
            r = rank[t, j]
            if r == 255:
                continue
            n = base[t] + r
            m = meta[t * 64 + j]
            assert nm_[n] == (m & 0x1ffffff) | (j << 25)
            w = nr[n]
            assert (w[3] >> 18) & 63 == r
            assert rec["unit_tile"][n >> 6] + ((w[3] >> 24) & 63) == t
            x, y, z = j & 3, (j >> 2) & 3, j >> 4
            for q in range(1, 19):
                if not (m >> q) & 1:      # bounce-back: the node's own rank
                    assert (w[(q - 1) // 5] >> (6 * ((q - 1) % 5))) & 63 == r
                    continue
                sx, sy, sz = x - e[q][0], y - e[q][1], z - e[q][2]
                d = [(-1 if v < 0 else (1 if v > 3 else 0)) for v in (sx, sy, sz)]
                kk = 9 * (d[0] + 1) + 3 * (d[1] + 1) + (d[2] + 1)
                src_t = t if kk == 13 else nbr[t, kk]
                src = (sx & 3) + 4 * (sy & 3) + 16 * (sz & 3)
                got = (w[(q - 1) // 5] >> (6 * ((q - 1) % 5))) & 63
                assert got == rank[src_t, src]
            checked += 1
    assert checked > 100

"""GPU parity at the BASELINE sizes ("next round" 1).

Tile maps (tiling.py:51-83): the device tiler's tile_map,
non_empty, neighbour rows, per-tile counts and every per-slot node word
(active / 18 pull links / tag / Zou-He face) equal the numpy oracle
(oracle/tiling.py) bit for bit on the config-3 sphere packs (256^3, 64
scan chunks), the config-4 vessel tree (512 x 512 x 1024, 4,096 chunks),
the periodic config-2 channel and ragged random media with inlet / outlet
on the x and y faces.

Fused step (boundaries.py:1-28): 10 steps of the GPU
solver against the C oracle (oracle/tlbm_oracle.c) from the same initial
state on the full config-2 channel 256^3 (fp64, fp32, fp64 FMA), the
config-3 packs at porosity 0.2 in both storages and both precisions, a
256 x 256 x 512 vessel tree and an MRT pack.

Tolerance (BASELINE.json north star), over non-solid nodes:
    rel(F) = max|F_gpu - F_oracle| / max|F_oracle|, F in {f, rho, u}
    fp64 <= 1e-12, fp32 <= 1e-5 (fp32 GPU vs the fp32 oracle).
Reference arithmetic is also asserted bit-exact; the FMA mode only within
the tolerance.
"""

import numpy as np
import pytest
import torch

from helpers import random_geometry
from oracle import tiling as ot
from oracle.numerics import E
from paper_1611_02445_b200 import geometry, tiling, workloads
from paper_1611_02445_b200.solver import SimulationConfig, Solver

pytestmark = pytest.mark.gpu
TOL = {"f64": 1e-12, "f32": 1e-5}


# ------------------------------------------------------------------ tiling
def _check_tiling(g):
    types = g.types
    grid = tiling.build_tiling(g)
    tm, ne = ot.build_tiling(types)
    assert grid.t_n == len(ne)
    assert np.array_equal(grid.tile_map, tm)
    assert np.array_equal(grid.non_empty, ne)
    nbr = ot.neighbor_indices(tm, ne, ot.DELTAS27, g.periodic)
    assert np.array_equal(grid.device.nbr.cpu().numpy(), nbr)
    meta = grid.device.meta.cpu().numpy()
    want = ot.meta_words(types, ne, g.periodic)
    assert np.array_equal(meta, want)
    counts = (want & 1).sum(1)
    assert np.array_equal(tiling.per_tile_nonsolid_counts(grid, g), counts)
    st = tiling.tile_utilization(grid, g)
    assert st.n_fn == int(np.count_nonzero(types)) == int(counts.sum())
    return grid


@pytest.mark.parametrize("porosity", [0.2, 0.5, 0.9])
def test_tiling_sphere_pack_256(porosity):
    """BASELINE config 3: 262,144 mesh tiles = 64 chunks of the device scan."""
    g = workloads.sphere_pack(porosity)
    grid = _check_tiling(g)
    assert grid.t_n < 64 ** 3              # sparse: the scan compacts across chunks


def test_tiling_vessel_tree_512x512x1024():
    """BASELINE config 4: 16.8 M mesh tiles, inlet z = 0, outlet z = 1023."""
    g = workloads.vessel_tree()
    assert (g.types == geometry.NodeType.VELOCITY_INLET).any()
    assert (g.types == geometry.NodeType.PRESSURE_OUTLET).any()
    _check_tiling(g)


def test_tiling_periodic_channel_256():
    """BASELINE config 2 (periodic z): wrap-around neighbour rows."""
    _check_tiling(workloads.channel_z(256))


@pytest.mark.parametrize("io_axis", [0, 1, 2])
def test_tiling_ragged_multichunk_io_faces(io_axis):
    """Ragged dims (not multiples of 4), ~100 k mesh tiles (25 chunks),
    inlet / outlet on the faces normal to ``io_axis``."""
    rng = np.random.default_rng(40 + io_axis)
    t = random_geometry(rng, (203, 118, 67), io_axis=io_axis)
    t[rng.random(t.shape) < 0.6] = 0          # sparse: many partly solid tiles
    g = geometry.Geometry(t, inlet_velocity=(0.01, 0.0, 0.0), outlet_density=1.0)
    _check_tiling(g)


# ------------------------------------------------------------------ fused step
def _dense(s):
    return s.to_dense(s.fields_canonical(device=True))


def _macro(f, quasi):
    """rho and u in the reference's order (collision.py:46-91)."""
    rho = f[0].clone()
    for q in range(1, 19):
        rho = rho + f[q]
    u = []
    for a in range(3):
        j = torch.zeros_like(rho)
        for q in range(1, 19):
            if E[q][a] == 1:
                j = j + f[q]
            elif E[q][a] == -1:
                j = j - f[q]
        u.append(j / rho if quasi else j)
    return rho, torch.stack(u)


def _rel(a, b):
    scale = b.abs().max()
    return float((a - b).abs().max() / (scale if scale > 0 else 1.0))


def _step_parity(c_oracle, s, geo, steps=10, exact=True):
    cfg = s.config
    prec = cfg.precision
    dt = np.float64 if prec == "f64" else np.float32
    f0 = _dense(s).cpu().numpy()
    op = cfg.mrt_operator
    o = c_oracle.DenseOracle(geo.types, cfg.fluid, cfg.tau, geo.inlet_velocity,
                             geo.outlet_density, periodic=geo.periodic, f0=f0, dtype=dt,
                             mrt_operator=None if op is None else np.asarray(op).astype(dt))
    assert o.run(steps) == 0
    s.step(steps)
    mask = torch.from_numpy(geo.types != 0).to(s.device)
    got = _dense(s)[:, mask]
    want = torch.from_numpy(o.f).to(s.device)[:, mask]
    del o
    quasi = getattr(cfg.fluid, "value", cfg.fluid) == "quasi-compressible"
    rg, ug = _macro(got, quasi)
    rw, uw = _macro(want, quasi)
    r = (_rel(got, want), _rel(rg, rw), _rel(ug, uw))
    assert max(r) <= TOL[prec], r
    if exact:
        assert torch.equal(got, want), f"not bit-exact: rel f/rho/u {r}"
    # the device rho/u readout (tlbm_macroscopic) equals the same reduction
    rho_d, u_d, _ = s.macroscopic(device=True)
    assert torch.equal(s.to_dense(rho_d)[mask], rg)
    assert torch.equal(s.to_dense(u_d)[:, mask], ug)
    return r


@pytest.mark.parametrize("prec,arith", [("f64", "reference"), ("f32", "reference"),
                                        ("f64", "fma")])
def test_step_channel_256(c_oracle, prec, arith):
    """BASELINE config 2, the bench workload: 256^3 channel periodic in z,
    perturbed equilibrium start (workloads.perturbed_fields), 10 steps."""
    geo = workloads.channel_z(256)
    s = workloads.make_solver(geo, prec, u0=(0.0, 0.0, 0.02), arithmetic=arith)
    r = _step_parity(c_oracle, s, geo, exact=arith == "reference")
    print(f"channel256 {prec} {arith}: rel f/rho/u = {r}")


@pytest.mark.parametrize("storage,traversal", [("blocks", "tile"), ("compact", "tile"),
                                               ("compact", "nodes")])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_step_sphere_pack_256_p02(c_oracle, prec, storage, traversal):
    """BASELINE config 3 at porosity 0.2 (tile utilisation 0.66), inlet z = 0 /
    outlet z = 255, both storages and both compact kernels (tile- and
    node-parallel), 10 steps from a perturbed start."""
    geo = workloads.sphere_pack(0.2)
    s = workloads.make_solver(geo, prec, u0=(0.0, 0.0, 0.01), storage=storage,
                              traversal=traversal)
    assert s.config.storage == storage and (s.nodes is not None) == (traversal == "nodes")
    _step_parity(c_oracle, s, geo)


def test_step_sphere_pack_256_p05_quasi_mrt(c_oracle):
    """Config 3 at porosity 0.5 with the secondary models: quasi-compressible
    fluid, MRT collision (collision.py:133-247), compact storage."""
    geo = workloads.sphere_pack(0.5)
    cfg = SimulationConfig(collision="mrt", fluid="quasi-compressible", tau=workloads.TAU,
                           precision="f64", storage="compact")
    s = Solver(geo, cfg)
    assert s.nodes is not None          # eta_t 0.825: the node-parallel step
    rho, u = workloads.perturbed_fields(s.t_n, s.store.tdtype, s.device, (0.0, 0.0, 0.01))
    s.init_from_macroscopic(rho, u)
    _step_parity(c_oracle, s, geo)


@pytest.mark.parametrize("geometry,storage", [("channel", "blocks"), ("pack02", "compact")])
def test_step_mrt_f32_full_size(c_oracle, geometry, storage):
    """fp32 MRT at BASELINE size, bit-exact vs the C oracle over 10 steps:
    the 256^3 channel on the block store (packed products and packed row
    sums, FFMA2(c, d, -0) + FADD2) and the porosity-0.2 pack on the compact
    store (node-parallel step, packed products only)."""
    geo = workloads.channel_z(256) if geometry == "channel" else workloads.sphere_pack(0.2)
    cfg = SimulationConfig(collision="mrt", tau=workloads.TAU, precision="f32",
                           storage=storage)
    s = Solver(geo, cfg)
    assert (s.nodes is not None) == (storage == "compact")
    rho, u = workloads.perturbed_fields(s.t_n, s.store.tdtype, s.device, (0.0, 0.0, 0.02))
    s.init_from_macroscopic(rho, u)
    _step_parity(c_oracle, s, geo)


@pytest.mark.parametrize("storage", ["blocks", "auto"])
def test_step_vessel_tree_256x256x512(c_oracle, storage):
    """BASELINE config 4 at half edge: velocity inlet z = 0, pressure outlet
    z = 511, bounce-back lumen shell, 10 steps from rest + inflow."""
    geo = workloads.vessel_tree((256, 256, 512))
    s = workloads.make_solver(geo, "f64", u0=(0.0, 0.0, 0.01), storage=storage)
    _step_parity(c_oracle, s, geo)


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("fluid", ["incompressible", "quasi-compressible"])
@pytest.mark.parametrize("io_axis", [0, 1])
def test_step_io_on_x_and_y_faces(c_oracle, io_axis, fluid, prec):
    """Zou-He inlet / outlet on the x and y faces (the z faces are covered
    above): ragged random media, 10 steps, bit-exact."""
    for seed in range(3):
        rng = np.random.default_rng(70 + 10 * io_axis + seed)
        shape = tuple(int(v) for v in rng.integers(6, 30, size=3))
        t = random_geometry(rng, shape, io_axis=io_axis)
        uin = [0.0, 0.0, 0.0]
        uin[io_axis] = 0.02
        uin[(io_axis + 1) % 3] = 0.005
        geo = geometry.Geometry(t, inlet_velocity=tuple(uin), outlet_density=1.002)
        cfg = SimulationConfig(fluid=fluid, tau=0.6, precision=prec, u_max_guard=0.0)
        s = Solver(geo, cfg)
        u0 = [0.0, 0.0, 0.0]
        u0[io_axis] = 0.01
        rho, u = workloads.perturbed_fields(s.t_n, s.store.tdtype, s.device, tuple(u0),
                                            seed=seed)
        s.init_from_macroscopic(rho, u)
        _step_parity(c_oracle, s, geo)


def test_step_io_faces_multichunk(c_oracle):
    """A ragged ~100 k-tile medium with inlet / outlet on the x faces and
    periodic y: the tiler's chunk carry, the Zou-He face code and the wrap
    together, fp64, 10 steps."""
    rng = np.random.default_rng(5)
    t = random_geometry(rng, (203, 120, 67), periodic=(False, True, False), io_axis=0)
    geo = geometry.Geometry(t, inlet_velocity=(0.02, 0.0, 0.0), outlet_density=1.0,
                            periodic=(False, True, False))
    s = workloads.make_solver(geo, "f64", u0=(0.01, 0.0, 0.0))
    _step_parity(c_oracle, s, geo)

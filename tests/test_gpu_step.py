"""GPU parity of the fused step against the CPU oracle and the reference.

Tolerance (BASELINE.json north star): rel(F) = max|F_gpu - F_oracle| /
max|F_oracle| over non-solid slots, F in {f (canonical), rho, u}:
    fp64 <= 1e-12, fp32 <= 1e-5   (fp32 GPU vs the fp32 oracle).
The kernel keeps the reference's operation order and no FMA contraction, so
the observed difference is 0 (bit-exact); the tests assert the stated
tolerance and, separately, bit-exactness where the arithmetic is identical.
"""

import warnings

import numpy as np
import pytest
import torch

from helpers import random_geometry
from oracle import dense, numerics as nm
from paper_1611_02445_b200 import _native as nat
from paper_1611_02445_b200 import collision, geometry, layout, solver

pytestmark = pytest.mark.gpu
MODELS = {"inc": collision.FluidModel.INCOMPRESSIBLE,
          "quasi": collision.FluidModel.QUASI_COMPRESSIBLE}
DTYPES = {"f64": np.float64, "f32": np.float32}
TOL = {np.float64: 1e-12, np.float32: 1e-5}


def rel(a, b):
    scale = np.abs(b).max()
    return float(np.abs(a - b).max() / (scale if scale else 1.0))


def make_solver(geo, model, dt, table=layout.LayoutTable.B200, tau=0.6, f0=None, guard=0.0):
    cfg = solver.SimulationConfig(fluid=model, tau=tau, precision="f64" if dt == np.float64
                                  else "f32", table=table, u_max_guard=guard)
    s = solver.Solver(geo, cfg)
    if f0 is not None:
        s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty,
                                                  f0.reshape(19, -1)[:, 0]))
    return s


def oracle_run(c_oracle, geo, model, dt, f0, steps, tau=0.6, mrt_operator=None):
    o = c_oracle.DenseOracle(geo.types, model, tau, geo.inlet_velocity, geo.outlet_density,
                             periodic=geo.periodic, f0=f0, dtype=dt,
                             mrt_operator=None if mrt_operator is None
                             else np.asarray(mrt_operator).astype(dt))
    o.run(steps)
    return o.f


def compare(s, f_dense, dt, exact=True):
    ne = s.tile_grid.non_empty
    want = dense.to_canonical(f_dense, ne, np.zeros(19))
    mask = s.nonsolid_mask()
    got = s.fields_canonical()
    g, w = got[:, mask], want[:, mask]
    r_f = rel(g, w)
    model = s.config.fluid
    rg, ug, _ = nm.macroscopic(model, g)
    rw, uw, _ = nm.macroscopic(model, w)
    r_rho, r_u = rel(rg, rw), rel(ug, uw)
    assert max(r_f, r_rho, r_u) <= TOL[dt], (r_f, r_rho, r_u)
    if exact:
        assert np.array_equal(g, w), f"not bit-exact (rel f {r_f:.3e})"
    # the device readout equals the oracle's macroscopic of the device fields
    rho_d, u_d, _ = s.macroscopic()
    assert np.array_equal(rho_d[mask], rg) and np.array_equal(u_d[:, mask], ug)
    return r_f, r_rho, r_u


def perturbed_eq(shape, model, dt, u=(0.0, 0.0, 0.0), seed=0, amp=1e-3):
    rng = np.random.default_rng(seed)
    f0 = dense.init_equilibrium(shape, model, dt, 1.0, u)
    return f0 * (1 + rng.uniform(-amp, amp, f0.shape)).astype(dt)


@pytest.mark.parametrize("table", list(layout.LayoutTable))
@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_reference_composed_golden(golden, table, dn, mn):
    """6 steps on a sphere pack with inlet/outlet == the step composed of the
    reference's own functions (tests/golden/make_golden.py)."""
    g = golden("step")
    dt, m = DTYPES[dn], MODELS[mn]
    geo = geometry.Geometry(g["types"], tuple(g["inlet_velocity"]), float(g["outlet_density"]))
    shape = geo.shape
    rho = np.ones(shape, dtype=dt)
    u = np.zeros((3,) + shape, dtype=dt)
    u[2] = 0.01
    f0 = nm.equilibrium(m, rho, u) * (1 + g["pert"]).astype(dt)
    s = make_solver(geo, m, dt, table, f0=f0)
    s.step(6)
    compare(s, g[f"f6_{dn}_{mn}"], dt)


@pytest.mark.parametrize("dn", DTYPES)
def test_cavity64_1000_steps(c_oracle, dn):
    """BASELINE config 1: lid-driven cavity 64^3, LBGK incompressible,
    1000 steps, vs the C oracle."""
    dt = DTYPES[dn]
    geo = geometry.generate_cavity3d(64)
    m = collision.FluidModel.INCOMPRESSIBLE
    f0 = dense.init_equilibrium(geo.shape, m, dt)
    s = make_solver(geo, m, dt)
    s.run(1000)
    want = oracle_run(c_oracle, geo, m, dt, f0, 1000)
    r = compare(s, want, dt)
    print(f"cavity64 {dn} 1000 steps rel f/rho/u = {r}")


@pytest.mark.parametrize("seed", range(20))
def test_random_geometries_all_tables(c_oracle, seed):
    """SPEC acceptance 6: >= 20 random mixed solid/fluid/bounce-back geometries
    <= 24^3 with inlet/outlet faces, 10 steps, both collision models, both
    fluid models, every layout table, f64 (and f32): the tiled GPU step equals
    the dense oracle (bit-exact; the stated bound is 1e-13 / 1e-5)."""
    rng = np.random.default_rng(100 + seed)
    shape = tuple(int(v) for v in rng.integers(4, 25, size=3))
    t = random_geometry(rng, shape)
    geo = geometry.Geometry(t, inlet_velocity=(0.01, 0.0, 0.02), outlet_density=1.001)
    for dt in (np.float64, np.float32):
        for m in MODELS.values():
            f0 = perturbed_eq(shape, m, dt, (0.0, 0.0, 0.01), seed)
            for coll in ("lbgk", "mrt"):
                op = solver.SimulationConfig(collision="mrt").mrt_operator if coll == "mrt" \
                    else None
                want = oracle_run(c_oracle, geo, m, dt, f0, 10, mrt_operator=op)
                for table in layout.LayoutTable:
                    cfg = solver.SimulationConfig(collision=coll, fluid=m, tau=0.6,
                                                  precision="f64" if dt == np.float64
                                                  else "f32", table=table, u_max_guard=0.0,
                                                  mrt_matrix=op)
                    s = solver.Solver(geo, cfg)
                    s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty,
                                                              nm.W))
                    s.step(10)
                    compare(s, want, dt)


@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_periodic_channel(c_oracle, dn, mn):
    """BASELINE config 2 in miniature: square channel periodic along x."""
    dt, m = DTYPES[dn], MODELS[mn]
    geo = geometry.generate_channel("square", 14, axis=0, offsets=(1, 3), length=24,
                                    ends="periodic")
    f0 = perturbed_eq(geo.shape, m, dt, (0.05, 0.0, 0.0), 4)
    s = make_solver(geo, m, dt, f0=f0)
    s.step(40)
    compare(s, oracle_run(c_oracle, geo, m, dt, f0, 40), dt)


def test_io_channel_and_sphere_pack(c_oracle):
    for geo in (geometry.generate_channel("circle", 13, axis=1, offsets=(2, 1), length=19,
                                          ends="io", inlet_velocity=(0.0, 0.02, 0.0)),
                geometry.generate_sphere_pack(28, 8, 0.5, seed=1234,
                                              inlet_velocity=(0.0, 0.0, 0.01))):
        for m in MODELS.values():
            f0 = dense.init_equilibrium(geo.shape, m, np.float64)
            s = make_solver(geo, m, np.float64)
            s.step(30)
            compare(s, oracle_run(c_oracle, geo, m, np.float64, f0, 30), np.float64)


def test_layout_invariance_cavity48():
    """SPEC acceptance 7: every layout table gives bit-identical fields
    (cavity 48^3, 100 steps, f64)."""
    geo = geometry.generate_cavity3d(48)
    outs = []
    for table in layout.LayoutTable:
        s = make_solver(geo, MODELS["inc"], np.float64, table)
        s.run(100)
        outs.append(s.fields_canonical(device=True))
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


def test_determinism():
    geo = geometry.generate_sphere_pack(40, 10, 0.6, seed=5, inlet_velocity=(0, 0, 0.02))
    runs = []
    for _ in range(2):
        s = make_solver(geo, MODELS["quasi"], np.float64)
        s.run(50)
        runs.append(s.fields_canonical(device=True))
    assert torch.equal(runs[0], runs[1])


@pytest.mark.parametrize("mn", MODELS)
def test_sealed_box_mass_conservation(mn):
    """SPEC acceptance 8: sealed bounce-back box 32^3, 1000 steps, f64,
    relative total-mass drift <= 1e-10."""
    t = np.full((32, 32, 32), 2, np.uint8)
    t[1:-1, 1:-1, 1:-1] = 1
    t[12:20, 3:9, 14:30] = 0
    geo = geometry.Geometry(t)
    m = MODELS[mn]
    s = make_solver(geo, m, np.float64, f0=perturbed_eq(t.shape, m, np.float64, seed=9))
    m0 = s.total_mass()
    s.run(1000)
    assert abs(s.total_mass() - m0) / m0 <= 1e-10


def test_fixed_point():
    geo = geometry.generate_channel("circle", 15, axis=2, length=12, ends="wall")
    s = make_solver(geo, MODELS["inc"], np.float64)
    before = s.fields_canonical()
    s.run(100)
    mask = s.nonsolid_mask()
    assert np.abs(s.fields_canonical()[:, mask] - before[:, mask]).max() <= 1e-15


def test_divergence_reports_iteration():
    geo = geometry.Geometry(np.ones((8, 8, 8), np.uint8), periodic=(True, True, True))
    s = make_solver(geo, MODELS["inc"], np.float64)
    s.step(3)
    f = s.fields_canonical()
    f[:, 0, 5] = np.nan
    s.store.fill_canonical(s.parity, f)
    with pytest.raises(collision.DivergenceError) as ei:
        s.step(5)
    assert ei.value.iteration == 3


def test_guard_warning():
    geo = geometry.Geometry(np.ones((8, 8, 8), np.uint8), periodic=(True, True, True))
    s = make_solver(geo, MODELS["inc"], np.float64, guard=0.05)
    s.init_equilibrium(1.0, (0.08, 0.0, 0.0))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        s.step(2)
    assert s.guard_iterations == [0, 1]
    assert any(issubclass(x.category, solver.CompressibilityWarning) for x in w)


def test_bench_variants():
    """rw-only copies each node's own values; propagation-only == the
    oracle's gather (no collision) (SPEC.md:531-539 bench ladder)."""
    geo = geometry.generate_sphere_pack(24, 6, 0.6, seed=2, inlet_velocity=(0, 0, 0.01))
    f0 = perturbed_eq(geo.shape, MODELS["inc"], np.float64, seed=3)
    s = make_solver(geo, MODELS["inc"], np.float64, f0=f0)
    mask = s.nonsolid_mask()
    start = s.fields_canonical()
    s.step(1, variant=nat.READ_WRITE_ONLY)
    assert np.array_equal(s.fields_canonical()[:, mask], start[:, mask])
    s.step(1, variant=nat.PROPAGATION_ONLY)
    want = dense.to_canonical(dense.gather(f0, geo.types), s.tile_grid.non_empty, np.zeros(19))
    assert np.array_equal(s.fields_canonical()[:, mask], want[:, mask])


def test_spec_step_and_run_api():
    geo = geometry.generate_cavity3d(16)
    cfg = solver.SimulationConfig()
    st = solver.init_state(cfg, geo)
    assert st.iteration == 0 and st.parity == 0
    st = solver.step(st)
    assert st.iteration == 1 and st.parity == 1
    st2, diag = solver.run(cfg, geo, 0)
    assert diag["iterations"] == 0 and diag["n_fn"] == 16 ** 3
    w = np.asarray(nm.W)
    f = st2.solver.fields_canonical()
    assert np.array_equal(f, np.broadcast_to(w[:, None, None], f.shape))


# -- MRT (SPEC acceptance 8, 9) ---------------------------------

def mrt_config(model, dt, op=None, rates=None, table=layout.LayoutTable.B200):
    return solver.SimulationConfig(collision="mrt", fluid=model, tau=0.6,
                                   precision="f64" if dt == np.float64 else "f32",
                                   table=table, u_max_guard=0.0, mrt_relaxation=rates,
                                   mrt_matrix=op)


@pytest.mark.parametrize("table", list(layout.LayoutTable))
@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_mrt_reference_composed_golden(golden, table, dn, mn):
    g = golden("step")
    dt, m = DTYPES[dn], MODELS[mn]
    geo = geometry.Geometry(g["types"], tuple(g["inlet_velocity"]), float(g["outlet_density"]))
    rho = np.ones(geo.shape, dtype=dt)
    u = np.zeros((3,) + geo.shape, dtype=dt)
    u[2] = 0.01
    f0 = nm.equilibrium(m, rho, u) * (1 + g["pert"]).astype(dt)
    s = solver.Solver(geo, mrt_config(m, dt, op=golden("lattice")["mrt_op_0.6"], table=table))
    s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
    s.step(4)
    compare(s, g[f"mrt4_{dn}_{mn}"], dt)


@pytest.mark.parametrize("seed", range(3))
def test_mrt_random_geometries(c_oracle, seed):
    rng = np.random.default_rng(500 + seed)
    shape = tuple(int(v) for v in rng.integers(6, 22, size=3))
    t = random_geometry(rng, shape)
    geo = geometry.Geometry(t, inlet_velocity=(0.0, 0.01, 0.02), outlet_density=1.0)
    for dt in (np.float64, np.float32):
        for m in MODELS.values():
            cfg = mrt_config(m, dt)
            f0 = perturbed_eq(shape, m, dt, (0.0, 0.0, 0.01), seed)
            o = c_oracle.DenseOracle(t, m, 0.6, geo.inlet_velocity, 1.0, f0=f0, dtype=dt,
                                     mrt_operator=cfg.mrt_operator.astype(dt))
            o.run(8)
            s = solver.Solver(geo, cfg)
            s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
            s.step(8)
            compare(s, o.f, dt)


@pytest.mark.parametrize("case", ["tau0.537", "tau2.9", "broken", "rates"])
def test_mrt_grouped_and_dense_products(c_oracle, case):
    """The step runs the grouped MRT product when the operator has the
    compiled column pattern (csrc/mrt_pattern.cuh) and the dense one when it
    does not (one perturbed coefficient, custom moment rates); both bit-exact
    vs the oracle, both storages."""
    rng = np.random.default_rng(77)
    shape = (14, 11, 17)
    t = random_geometry(rng, shape)
    geo = geometry.Geometry(t, inlet_velocity=(0.0, 0.01, 0.02), outlet_density=1.0)
    tau = {"tau0.537": 0.537, "tau2.9": 2.9}.get(case, 0.6)
    rates = None
    op = None
    if case == "broken":
        op = solver.SimulationConfig(collision="mrt", tau=tau).mrt_operator.copy()
        op[4, 0] = np.nextafter(op[4, 0], 1.0)
    if case == "rates":
        rates = np.random.default_rng(3).uniform(0.8, 1.9, 19)
    for dt in (np.float64, np.float32):
        m = MODELS["inc"]
        for storage in ("blocks", "compact"):
            cfg = solver.SimulationConfig(collision="mrt", fluid=m, tau=tau, storage=storage,
                                          precision="f64" if dt == np.float64 else "f32",
                                          u_max_guard=0.0, mrt_relaxation=rates, mrt_matrix=op)
            f0 = perturbed_eq(shape, m, dt, (0.0, 0.0, 0.01), 9)
            o = c_oracle.DenseOracle(t, m, tau, geo.inlet_velocity, 1.0, f0=f0, dtype=dt,
                                     mrt_operator=cfg.mrt_operator.astype(dt))
            o.run(6)
            s = solver.Solver(geo, cfg)
            s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
            s.step(6)
            compare(s, o.f, dt)


def test_mrt_bgk_limit():
    """SPEC acceptance 9: all moment rates = 1/tau -> MRT == LBGK to 1e-12."""
    geo = geometry.generate_sphere_pack(24, 6, 0.6, seed=8, inlet_velocity=(0, 0, 0.01))
    m = MODELS["inc"]
    f0 = perturbed_eq(geo.shape, m, np.float64, (0.0, 0.0, 0.01), 4)
    runs = []
    for coll in ("lbgk", "mrt"):
        cfg = solver.SimulationConfig(collision=coll, tau=0.6, u_max_guard=0.0,
                                      mrt_relaxation=np.full(19, 1 / 0.6))
        s = solver.Solver(geo, cfg)
        s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
        s.step(10)
        runs.append(s.fields_canonical()[:, s.nonsolid_mask()])
    assert rel(runs[1], runs[0]) <= 1e-12


@pytest.mark.parametrize("mn", MODELS)
def test_mrt_sealed_box_mass_conservation(mn):
    t = np.full((32, 32, 32), 2, np.uint8)
    t[1:-1, 1:-1, 1:-1] = 1
    t[12:20, 3:9, 14:30] = 0
    geo = geometry.Geometry(t)
    m = MODELS[mn]
    s = solver.Solver(geo, mrt_config(m, np.float64))
    s.set_fields_canonical(dense.to_canonical(perturbed_eq(t.shape, m, np.float64, seed=9),
                                              s.tile_grid.non_empty, nm.W))
    m0 = s.total_mass()
    s.run(1000)
    assert abs(s.total_mass() - m0) / m0 <= 1e-10


@pytest.mark.parametrize("coll", ["lbgk", "mrt"])
def test_index64_path(c_oracle, coll):
    """The 64-bit addressing variant (domains beyond ~1.76 M tiles) forced on a
    small geometry: same bits as the oracle."""
    geo = geometry.generate_sphere_pack(30, 8, 0.55, seed=21, inlet_velocity=(0, 0, 0.02))
    for dt in (np.float64, np.float32):
        for m in MODELS.values():
            op = solver.SimulationConfig(collision="mrt").mrt_operator if coll == "mrt" else None
            f0 = perturbed_eq(geo.shape, m, dt, (0.0, 0.0, 0.01), 7)
            want = oracle_run(c_oracle, geo, m, dt, f0, 12, mrt_operator=op)
            cfg = solver.SimulationConfig(collision=coll, fluid=m, tau=0.6, u_max_guard=0.0,
                                          precision="f64" if dt == np.float64 else "f32",
                                          mrt_matrix=op)
            s = solver.Solver(geo, cfg, index64=True)
            assert s._args.rel32 == 0
            s.set_fields_canonical(dense.to_canonical(f0, s.tile_grid.non_empty, nm.W))
            s.step(12)
            compare(s, want, dt)


@pytest.mark.parametrize("storage", ["blocks", "compact"])
@pytest.mark.parametrize("dn", DTYPES)
def test_blocked_traversal_bit_identical(storage, dn):
    """The y-blocked visiting order (Solver(traversal=yb)) only reorders the
    independent tile updates: results equal the tile-list order."""
    geo = geometry.generate_sphere_pack(40, 10, 0.5, seed=13, inlet_velocity=(0, 0, 0.02))
    runs = []
    for trav in ("tile", 2):
        cfg = solver.SimulationConfig(precision=dn, u_max_guard=0.0, storage=storage)
        s = solver.Solver(geo, cfg, traversal=trav)
        assert (s.order is None) == (trav == "tile")
        s.init_equilibrium(1.0, (0.0, 0.0, 0.01))
        s.step(70, graph=True)
        runs.append(s.fields_canonical(device=True))
    assert torch.equal(runs[0], runs[1])
    if True:
        order = solver.traversal_order(s.tiling, s.store, 2)
        assert torch.equal(torch.sort(order.long()).values,
                           torch.arange(s.t_n, device=order.device))


@pytest.mark.parametrize("storage,traversal", [("blocks", "tile"), ("compact", "tile"),
                                               ("compact", "nodes")])
def test_degenerate_geometries(storage, traversal):
    """All-solid (no tiles) and single-node geometries step, graph-replay,
    read out and checkpoint without errors (both compact kernels)."""
    import tempfile
    cfg = solver.SimulationConfig(u_max_guard=0.0, storage=storage)
    empty = geometry.Geometry(np.zeros((5, 6, 7), np.uint8))
    s = solver.Solver(empty, cfg, traversal=traversal)
    assert s.t_n == 0 and s.n_fn == 0
    s.step(3)
    s.step(solver.GRAPH_STEPS, graph=True)
    rho, u, p = s.macroscopic()
    assert rho.shape == (0, 64) and u.shape == (3, 0, 64)
    one = np.zeros((3, 3, 3), np.uint8)
    one[1, 1, 1] = 1                        # a single fluid node, fully enclosed
    s = solver.Solver(geometry.Geometry(one), cfg, traversal=traversal)
    assert (s.nodes is not None) == (traversal == "nodes")
    s.step(10)
    rho, _, _ = s.macroscopic()
    assert abs(rho[s.nonsolid_mask()][0] - 1.0) < 1e-15
    with tempfile.TemporaryDirectory() as d:
        s.save_checkpoint(d + "/ck.npz")
        assert solver.resume(d + "/ck.npz", geometry.Geometry(one)).iteration == 10

"""GPU: node physics kernels and the field store, bit-exact vs the reference
(golden vectors from tests/golden/make_golden.py)."""

import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle import tiling as ot
from paper_1611_02445_b200 import boundaries, collision, geometry, layout, solver

pytestmark = pytest.mark.gpu
MODELS = {"inc": collision.FluidModel.INCOMPRESSIBLE,
          "quasi": collision.FluidModel.QUASI_COMPRESSIBLE}
DTYPES = {"f64": np.float64, "f32": np.float32}


@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_collision_kernels_golden(golden, dn, mn):
    g = golden("numerics")
    f = g[f"f_{dn}"]
    m = MODELS[mn]
    rho, u, p = collision.macroscopic(m, f)
    assert rho.dtype == f.dtype
    assert np.array_equal(rho, g[f"rho_{dn}_{mn}"])
    assert np.array_equal(u, g[f"u_{dn}_{mn}"])
    assert np.array_equal(p, g[f"p_{dn}_{mn}"])
    assert np.array_equal(collision.equilibrium(m, rho, u), g[f"feq_{dn}_{mn}"])
    assert np.array_equal(collision.collide_lbgk(m, f, 0.6), g[f"post_{dn}_{mn}"])
    # torch tensors stay on the device
    ft = torch.from_numpy(f).cuda()
    r2, _, _ = collision.macroscopic(m, ft)
    assert r2.is_cuda and np.array_equal(r2.cpu().numpy(), g[f"rho_{dn}_{mn}"])


@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_zou_he_kernels_golden(golden, dn, mn):
    g = golden("numerics")
    f = g[f"f_{dn}"]
    m = MODELS[mn]
    for (axis, sign), c in boundaries.FACE_CLOSURES.items():
        key = f"{axis}{'lo' if sign > 0 else 'hi'}"
        h = f.copy()
        r = boundaries.zou_he_velocity(h, c, (0.03, -0.02, 0.01), m)
        assert np.array_equal(h, g[f"zhv_{dn}_{mn}_{key}"]), key
        assert np.array_equal(r, g[f"zhv_ret_{dn}_{mn}_{key}"]), key
        h = f.copy()
        r = boundaries.zou_he_pressure(h, c, 1.02, m)
        assert np.array_equal(h, g[f"zhp_{dn}_{mn}_{key}"]), key
        assert np.array_equal(r, g[f"zhp_ret_{dn}_{mn}_{key}"]), key


def test_quasi_divergence_raises():
    f = np.zeros((19, 4))
    with pytest.raises(collision.DivergenceError):
        collision.macroscopic(collision.FluidModel.QUASI_COMPRESSIBLE, f)


def test_reflect_density_momentum():
    rng = np.random.default_rng(0)
    f = rng.random((19, 7))
    assert np.array_equal(collision.reflect(f), f[nm.OPP])
    assert np.array_equal(collision.density(f), nm.density(f))
    assert np.array_equal(collision.momentum(f), nm.momentum(f))


@pytest.mark.parametrize("table", list(layout.LayoutTable))
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_field_store_roundtrip(table, dt):
    rng = np.random.default_rng(1)
    t_n = 37
    vals = rng.standard_normal((19, t_n, 64)).astype(dt)
    fs = layout.FieldStore(t_n, table, dt)
    fs.fill_canonical(1, vals)
    assert np.array_equal(fs.read_canonical(1), vals)
    # stored order follows the table's permutations (layout.py:155-159)
    blocks = fs.blocks(1).cpu().numpy()
    assert np.array_equal(blocks, ot.to_blocks(vals, table.value))
    flat = fs.flat.cpu().numpy()
    addr = layout.value_address(5, 8, 1, 3, 1, 2, t_n=t_n, table=table)
    assert flat[addr] == vals[8, 5, 3 + 4 * 1 + 16 * 2]


@pytest.mark.parametrize("mn", MODELS)
def test_init_from_macroscopic(mn):
    rng = np.random.default_rng(2)
    g = geometry.generate_cavity3d(12)
    s = solver.Solver(g, solver.SimulationConfig(fluid=MODELS[mn]))
    rho = 1 + 1e-3 * rng.standard_normal((s.t_n, 64))
    u = 1e-2 * rng.standard_normal((3, s.t_n, 64))
    s.init_from_macroscopic(rho, u)
    want = nm.equilibrium(MODELS[mn], rho, u)
    for c in (0, 1):
        assert np.array_equal(s.fields_canonical(copy=c), want)
    r2, u2, p2 = s.macroscopic()
    assert np.array_equal((r2, u2, p2)[0], nm.macroscopic(MODELS[mn], want)[0])
    assert np.array_equal(u2, nm.macroscopic(MODELS[mn], want)[1])


@pytest.mark.parametrize("dn", DTYPES)
@pytest.mark.parametrize("mn", MODELS)
def test_collide_mrt_golden(golden, dn, mn):
    g = golden("numerics")
    f = g[f"f_{dn}"]
    op = golden("lattice")["mrt_op_0.6"]
    # the golden is collide_mrt(rates=...): operator built in float64 and
    # rounded to f's dtype (collision.py:241-243)
    for kw in ({"rates": collision.default_mrt_rates(0.6)}, {"operator": op.astype(f.dtype)}):
        out = collision.collide_mrt(MODELS[mn], f, **kw)
        assert out.dtype == f.dtype
        assert np.array_equal(out, g[f"mrt_{dn}_{mn}"])


@pytest.mark.parametrize("mn", MODELS)
def test_collide_mrt_float64_operator_on_float32(golden, mn):
    """An explicit float64 operator on float32 populations follows NumPy's
    promotion: each c * delta term in float64, rounded into the
    float32 accumulator -- the oracle's numpy restatement of collision.py:
    216-247 on the same inputs, bit for bit."""
    from oracle import numerics as onm
    g = golden("numerics")
    f = g["f_f32"]
    op = golden("lattice")["mrt_op_0.6"]
    assert op.dtype == np.float64
    want = onm.collide_mrt(MODELS[mn].value, f, operator=op)
    assert want.dtype == np.float32
    got = collision.collide_mrt(MODELS[mn], f, operator=op)
    assert got.dtype == np.float32 and np.array_equal(got, want)
    # and it differs from the operator rounded to float32 first
    narrow = collision.collide_mrt(MODELS[mn], f, operator=op.astype(np.float32))
    assert not np.array_equal(narrow, want)


def test_mrt_setup_matches_oracle(golden):
    g = golden("lattice")
    assert np.array_equal(collision.MOMENT_MATRIX, g["moments"])
    assert np.array_equal(collision.default_mrt_rates(0.6), g["mrt_rates_0.6"])
    assert np.allclose(collision.mrt_operator(collision.default_mrt_rates(0.6)),
                       g["mrt_op_0.6"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("dn", ["f64", "f32"])
def test_apply_operator_golden(golden, dn):
    """collision.apply_operator == the reference's fixed-order, zero-skipping
    accumulation (collision.py:216-231), bit for bit (numpy reference run in
    the test on the same inputs)."""
    import numpy as np
    from paper_1611_02445_b200 import collision
    dt = np.float64 if dn == "f64" else np.float32
    rng = np.random.default_rng(4)
    op = golden("lattice")["mrt_op_0.6"].copy()
    op[3, 5] = 0.0                                   # exercise the zero skip
    for op_dt in (np.float64, dt):
        opx = op.astype(op_dt)
        d = (rng.standard_normal((19, 7, 5)) * 1e-3).astype(dt)
        want = np.empty_like(d)
        for i in range(19):
            acc = np.zeros_like(d[0])
            for j in range(19):
                if opx[i, j] != 0.0:
                    acc += opx[i, j] * d[j]
            want[i] = acc
        got = collision.apply_operator(opx, d)
        assert got.dtype == d.dtype and np.array_equal(got, want)

"""Generate the golden vectors in tests/golden/ from the REFERENCE itself.

Run in the dev container (needs /root/reference):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Everything here calls the reference package ``tilelbm`` (imported from
/root/reference/pkg/src), never this repo's code:

* lattice.npz   -- E_VECTORS, WEIGHTS, OPPOSITE, table_permutations
                   (layout.py:108-112) for both reference tables.
* numerics.npz  -- macroscopic / equilibrium / collide_lbgk (collision.py)
                   and zou_he_velocity / zou_he_pressure (boundaries.py) on
                   seeded random populations, f64 and f32, both fluid models,
                   all six faces.
* tiling.npz    -- build_tiling (tiling.py:51-83), _neighbor_indices over the
                   27 deltas and _tile_nonsolid_blocks (txmodel.py:145-173) of
                   reference-generated geometries (cavity, channels, packs).
* faces.npz     -- classify_boundary_faces (boundaries.py:95-129) on
                   reference-generated geometries with inlet/outlet on the
                   x, y and z faces and a box with both kinds on all six
                   faces; tile_utilization (tiling.py:120-140) statistics.
* step.npz      -- the step has no reference implementation, so
                   it is composed here from reference functions only
                   (classify_boundary_faces, FACE_CLOSURES, zou_he_*,
                   collide_lbgk / collide_mrt, reflect) following SURVEY
                   Appendix A: a small sphere pack with inlet/outlet, 6 LBGK
                   steps and 4 MRT steps (default rates), f64/f32, both fluid
                   models.  Pins the oracle and the GPU step to reference
                   arithmetic.
"""

import itertools
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from tilelbm import boundaries as rb  # noqa: E402
from tilelbm import collision as rc  # noqa: E402
from tilelbm import geometry as rg  # noqa: E402
from tilelbm import lattice as rl  # noqa: E402
from tilelbm import layout as rlay  # noqa: E402
from tilelbm import tiling as rt  # noqa: E402
from tilelbm import txmodel as rx  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MODELS = {"inc": rc.FluidModel.INCOMPRESSIBLE, "quasi": rc.FluidModel.QUASI_COMPRESSIBLE}
DTYPES = {"f64": np.float64, "f32": np.float32}


def lattice():
    out = {"e": rl.E_VECTORS, "w": rl.WEIGHTS, "opp": rl.OPPOSITE,
           "moments": rc.MOMENT_MATRIX, "mrt_rates_0.6": rc.default_mrt_rates(0.6),
           "mrt_op_0.6": rc.mrt_operator(rc.default_mrt_rates(0.6))}
    for t in rlay.LayoutTable:
        out[f"perm_{t.value}"] = rlay.table_permutations(t)
    np.savez_compressed(os.path.join(HERE, "lattice.npz"), **out)


def numerics():
    rng = np.random.default_rng(20161107)
    out = {}
    for dn, dt in DTYPES.items():
        f = (rl.WEIGHTS[:, None] * rng.uniform(0.8, 1.2, (19, 16))).astype(dt)
        out[f"f_{dn}"] = f
        for mn, m in MODELS.items():
            rho, u, p = rc.macroscopic(m, f)
            out[f"rho_{dn}_{mn}"], out[f"u_{dn}_{mn}"], out[f"p_{dn}_{mn}"] = rho, u, p
            out[f"feq_{dn}_{mn}"] = rc.equilibrium(m, rho, u)
            out[f"post_{dn}_{mn}"] = rc.collide_lbgk(m, f, 0.6)
            out[f"mrt_{dn}_{mn}"] = rc.collide_mrt(m, f, rates=rc.default_mrt_rates(0.6))
            for (axis, sign), c in rb.FACE_CLOSURES.items():
                key = f"{axis}{'lo' if sign > 0 else 'hi'}"
                g = f.copy()
                out[f"zhv_ret_{dn}_{mn}_{key}"] = rb.zou_he_velocity(g, c, (0.03, -0.02, 0.01), m)
                out[f"zhv_{dn}_{mn}_{key}"] = g
                g = f.copy()
                out[f"zhp_ret_{dn}_{mn}_{key}"] = rb.zou_he_pressure(g, c, 1.02, m)
                out[f"zhp_{dn}_{mn}_{key}"] = g
    np.savez_compressed(os.path.join(HERE, "numerics.npz"), **out)


def tiling_cases():
    return {
        "cavity10": rg.generate_cavity3d(10),
        "cavity13": rg.generate_cavity3d(13),
        "chan_sq": rg.generate_channel("square", 9, axis=1, offsets=(1, 2), length=11),
        "chan_ci": rg.generate_channel("circle", 10, axis=2, offsets=(3, 1), length=9,
                                       ends="io"),
        "pack": rg.generate_sphere_pack(22, 8, 0.55, seed=7),
        "pack_x": rg.generate_sphere_pack(17, 6, 0.7, seed=3, flow_axis=0),
    }


def tiling():
    out = {}
    deltas = list(itertools.product((-1, 0, 1), repeat=3))
    for name, g in tiling_cases().items():
        grid = rt.build_tiling(g)
        out[f"{name}_types"] = g.types
        out[f"{name}_tile_map"] = grid.tile_map
        out[f"{name}_non_empty"] = grid.non_empty
        out[f"{name}_nbr"] = rx._neighbor_indices(grid, deltas)
        out[f"{name}_nonsolid"] = rx._tile_nonsolid_blocks(grid, g)
        out[f"{name}_counts"] = rt.per_tile_nonsolid_counts(grid, g)
    np.savez_compressed(os.path.join(HERE, "tiling.npz"), **out)


def reference_step(f, geometry, model, tau, mrt=False):
    """One step composed only of reference functions."""
    t = geometry.types
    nx, ny, nz = t.shape
    ns = t != rg.NodeType.SOLID
    g = np.empty_like(f)
    g[0] = f[0]
    for q in range(1, 19):
        e = rl.E_VECTORS[q]
        src_val = np.zeros_like(f[q])
        src_ok = np.zeros(t.shape, dtype=bool)
        dst = tuple(slice(max(0, int(c)), n + min(0, int(c))) for c, n in zip(e, t.shape))
        src = tuple(slice(max(0, -int(c)), n - max(0, int(c))) for c, n in zip(e, t.shape))
        src_val[dst] = f[q][src]
        src_ok[dst] = ns[src]
        g[q] = np.where(src_ok, src_val, f[rl.OPPOSITE[q]])
    if mrt:
        op = rc.mrt_operator(rc.default_mrt_rates(tau), dtype=f.dtype)
        collide = lambda h: rc.collide_mrt(model, h, operator=op)  # noqa: E731
    else:
        collide = lambda h: rc.collide_lbgk(model, h, tau)  # noqa: E731
    new = f.copy()
    fl = t == rg.NodeType.FLUID
    new[:, fl] = collide(g[:, fl])
    bb = t == rg.NodeType.BB_WALL
    new[:, bb] = rc.reflect(g[:, bb])
    for key, (inlet, outlet) in rb.classify_boundary_faces(geometry).items():
        c = rb.FACE_CLOSURES[key]
        for ids, is_in in ((inlet, True), (outlet, False)):
            if ids.size == 0:
                continue
            idx = np.unravel_index(ids, t.shape)
            sub = g[(slice(None),) + idx].copy()
            if is_in:
                rb.zou_he_velocity(sub, c, geometry.inlet_velocity, model)
            else:
                rb.zou_he_pressure(sub, c, geometry.outlet_density, model)
            new[(slice(None),) + idx] = collide(sub)
    return new


def step():
    out = {}
    geo = rg.generate_sphere_pack(10, 4, 0.6, seed=11, inlet_velocity=(0.0, 0.0, 0.02),
                                  outlet_density=1.0)
    out["types"] = geo.types
    out["inlet_velocity"] = np.array(geo.inlet_velocity)
    out["outlet_density"] = np.array(geo.outlet_density)
    rng = np.random.default_rng(99)
    pert = rng.uniform(-1e-3, 1e-3, (19,) + geo.shape)
    out["pert"] = pert
    for dn, dt in DTYPES.items():
        for mn, m in MODELS.items():
            rho = np.ones(geo.shape, dtype=dt)
            u = np.zeros((3,) + geo.shape, dtype=dt)
            u[2] = 0.01
            # f0 = equilibrium(1, (0, 0, 0.01)) * (1 + pert), rebuilt by the tests
            f0 = rc.equilibrium(m, rho, u) * (1 + pert).astype(dt)
            f = f0
            for _ in range(6):
                f = reference_step(f, geo, m, 0.6)
            out[f"f6_{dn}_{mn}"] = f
            f = f0
            for _ in range(4):
                f = reference_step(f, geo, m, 0.6, mrt=True)
            out[f"mrt4_{dn}_{mn}"] = f
    np.savez_compressed(os.path.join(HERE, "step.npz"), **out)


def six_face_box():
    """Interior FLUID box whose six faces carry inlets (low faces) and
    outlets (high faces) inside a bounce-back rim, plus a few interior
    solids and walls."""
    t = np.ones((12, 10, 9), dtype=np.uint8)
    for a in range(3):
        lo = [slice(None)] * 3
        hi = [slice(None)] * 3
        lo[a], hi[a] = 0, -1
        t[tuple(lo)] = rg.NodeType.VELOCITY_INLET
        t[tuple(hi)] = rg.NodeType.PRESSURE_OUTLET
    # edges and corners (on two or three faces) -> bounce-back rim
    x, y, z = np.meshgrid(*(np.arange(n) for n in t.shape), indexing="ij")
    on = sum(((c == 0) | (c == n - 1)).astype(int) for c, n in zip((x, y, z), t.shape))
    t[on >= 2] = rg.NodeType.BB_WALL
    t[5, 4, 4] = rg.NodeType.SOLID
    t[6, 5, 3] = rg.NodeType.BB_WALL
    t[0, 3, 3] = rg.NodeType.SOLID           # a hole in the x-low inlet plane
    t[11, 4, 6] = rg.NodeType.BB_WALL        # a wall node in the x-high outlet plane
    return rg.Geometry(t, inlet_velocity=(0.01, 0.0, 0.0), outlet_density=1.0)


def face_cases():
    return {
        "cavity10": rg.generate_cavity3d(10),
        "chan_io_z": rg.generate_channel("circle", 10, axis=2, offsets=(3, 1), length=9,
                                         ends="io"),
        "chan_io_x": rg.generate_channel("square", 8, axis=0, offsets=(1, 1), length=13,
                                         ends="io", inlet_velocity=(0.02, 0.0, 0.0)),
        "chan_io_y": rg.generate_channel("circle", 9, axis=1, offsets=(2, 1), length=7,
                                         ends="io", inlet_velocity=(0.0, 0.02, 0.0)),
        "pack_z": rg.generate_sphere_pack(22, 8, 0.55, seed=7),
        "pack_x": rg.generate_sphere_pack(17, 6, 0.7, seed=3, flow_axis=0),
        "pack_y": rg.generate_sphere_pack(19, 6, 0.6, seed=5, flow_axis=1),
        "box6": six_face_box(),
    }


def faces():
    out = {}
    for name, g in face_cases().items():
        out[f"{name}_types"] = g.types
        res = rb.classify_boundary_faces(g)
        out[f"{name}_keys"] = np.array(sorted(res), dtype=np.int64).reshape(-1, 2)
        for (axis, sign), (inlet, outlet) in res.items():
            out[f"{name}_{axis}_{sign}_in"] = inlet
            out[f"{name}_{axis}_{sign}_out"] = outlet
        st = rt.tile_utilization(rt.build_tiling(g), g)
        out[f"{name}_util"] = np.array([st.t_n, st.n_fn, st.eta_t, st.n_tfn, st.n_tsn,
                                        st.eta_f, st.eta_e], dtype=np.float64)
    # rejected: an inlet on a corner (three faces) and an outlet inside
    bad = np.ones((6, 6, 6), dtype=np.uint8)
    bad[0, 0, 0] = rg.NodeType.VELOCITY_INLET
    out["bad_corner_types"] = bad
    bad = np.ones((6, 6, 6), dtype=np.uint8)
    bad[2, 3, 3] = rg.NodeType.PRESSURE_OUTLET
    out["bad_interior_types"] = bad
    for k in ("bad_corner", "bad_interior"):
        try:
            rb.classify_boundary_faces(rg.Geometry(out[f"{k}_types"]))
            raise AssertionError("reference accepted a misplaced inlet/outlet")
        except ValueError as exc:
            out[f"{k}_msg"] = np.array(str(exc))
    np.savez_compressed(os.path.join(HERE, "faces.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:                      # regenerate selected files only
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    lattice()
    numerics()
    tiling()
    faces()
    step()
    print("golden vectors written to", HERE)

"""GPU: the device tiler is bit-exact with the reference's build_tiling,
_neighbor_indices and per-tile counts (golden vectors made by the reference,
plus the oracle restatement on further geometries)."""

import itertools

import numpy as np
import pytest

from oracle import tiling as ot
from paper_1611_02445_b200 import geometry as geo_mod
from paper_1611_02445_b200 import tiling

pytestmark = pytest.mark.gpu
D27 = list(itertools.product((-1, 0, 1), repeat=3))


def _check(g, types, tm_ref, ne_ref, nbr_ref=None, counts_ref=None, periodic=(False,) * 3):
    grid = tiling.build_tiling(g)
    assert grid.tile_map.dtype == np.int32 and grid.non_empty.dtype == np.int32
    assert np.array_equal(grid.tile_map, tm_ref)
    assert np.array_equal(grid.non_empty, ne_ref)
    if nbr_ref is None:
        nbr_ref = ot.neighbor_indices(tm_ref, ne_ref, D27, periodic)
    assert np.array_equal(grid.device.nbr.cpu().numpy(), nbr_ref)
    if counts_ref is None:
        counts_ref = ot.nonsolid_blocks(types, ne_ref).sum(1)
    assert np.array_equal(tiling.per_tile_nonsolid_counts(grid, g), counts_ref)
    meta = grid.device.meta.cpu().numpy()
    assert np.array_equal((meta & 1).astype(bool), ot.nonsolid_blocks(types, ne_ref))
    assert np.array_equal((meta >> 19) & 7, ot.tile_types(types, ne_ref))
    return grid


def test_golden_tilings(golden):
    gd = golden("tiling")
    names = sorted({k.rsplit("_", 1)[0] for k in gd if k.endswith("_types")})
    for name in names:
        types = gd[f"{name}_types"]
        g = geo_mod.Geometry(types)
        _check(g, types, gd[f"{name}_tile_map"], gd[f"{name}_non_empty"], gd[f"{name}_nbr"],
               gd[f"{name}_counts"])


@pytest.mark.parametrize("shape", [(4, 4, 4), (5, 9, 3), (1, 1, 1), (33, 17, 21), (64, 8, 130)])
def test_random_tilings(shape):
    rng = np.random.default_rng(sum(shape))
    for density in (0.02, 0.3, 0.9):
        types = (rng.random(shape) < density).astype(np.uint8)
        g = geo_mod.Geometry(types)
        tm, ne = ot.build_tiling(types)
        if len(ne) == 0:
            grid = tiling.build_tiling(g)
            assert grid.t_n == 0 and np.all(grid.tile_map == -1)
            continue
        _check(g, types, tm, ne)


def test_all_solid():
    grid = tiling.build_tiling(geo_mod.Geometry(np.zeros((9, 4, 6), np.uint8)))
    assert grid.t_n == 0
    assert grid.tile_map.shape == (3, 1, 2) and np.all(grid.tile_map == -1)


def test_cavity100_tile_count():
    """SPEC tiling example: cavity3d(100) -> t_n = 25^3 = 15625."""
    g = geo_mod.generate_cavity3d(100)
    grid = tiling.build_tiling(g)
    assert grid.t_n == 15625
    st = tiling.tile_utilization(grid, g)
    assert st.n_fn == 100 ** 3 and st.eta_t == 1.0


def test_periodic_neighbors():
    g = geo_mod.generate_channel("square", 12, axis=0, length=16, ends="periodic")
    types = g.types
    tm, ne = ot.build_tiling(types)
    _check(g, types, tm, ne, periodic=g.periodic)


def test_sphere_pack_counts():
    g = geo_mod.generate_sphere_pack(48, 12, 0.5, seed=1234)
    types = g.types
    tm, ne = ot.build_tiling(types)
    grid = _check(g, types, tm, ne)
    st = tiling.tile_utilization(grid, g)
    assert st.n_fn == g.nonsolid_count()


FACE_CASES = ("cavity10", "chan_io_z", "chan_io_x", "chan_io_y", "pack_z", "pack_x", "pack_y",
              "box6")


@pytest.mark.parametrize("name", FACE_CASES)
def test_utilization_golden(golden, name):
    """tile_utilization (tiling.py:120-140) == the reference's statistics
    (tests/golden/faces.npz, made by the reference), exactly."""
    gd = golden("faces")
    g = geo_mod.Geometry(gd[f"{name}_types"])
    st = tiling.tile_utilization(tiling.build_tiling(g), g)
    want = gd[f"{name}_util"]
    assert (st.t_n, st.n_fn) == (int(want[0]), int(want[1]))
    assert np.array_equal(np.array([st.eta_t, st.n_tfn, st.n_tsn, st.eta_f, st.eta_e]),
                          want[2:])


@pytest.mark.parametrize("name", FACE_CASES)
def test_classify_boundary_faces_golden(golden, name):
    """boundaries.classify_boundary_faces (boundaries.py:95-129) == the
    reference's output: same keys, same flat C-order inlet / outlet ids,
    on x, y and z faces and all six faces of one box; and the device node
    words carry the same face code for every inlet / outlet slot."""
    from paper_1611_02445_b200 import boundaries
    gd = golden("faces")
    types = gd[f"{name}_types"]
    g = geo_mod.Geometry(types)
    got = boundaries.classify_boundary_faces(g)
    keys = [(int(a), int(s)) for a, s in gd[f"{name}_keys"]]
    assert sorted(got) == sorted(keys)
    face = np.full(types.size, -1, dtype=np.int64)
    for a, s in keys:
        inl, outl = got[(a, s)]
        assert np.array_equal(inl, gd[f"{name}_{a}_{s}_in"])
        assert np.array_equal(outl, gd[f"{name}_{a}_{s}_out"])
        assert boundaries.FACE_CLOSURES[(a, s)].face_id == 2 * a + (0 if s > 0 else 1)
        face[inl] = face[outl] = 2 * a + (0 if s > 0 else 1)
    grid = tiling.build_tiling(g)
    meta = grid.device.meta.cpu().numpy().astype(np.int64)
    ne = grid.non_empty
    j = np.arange(64)
    x, y, z = ne[:, 0:1] + (j & 3), ne[:, 1:2] + ((j >> 2) & 3), ne[:, 2:3] + (j >> 4)
    nx, ny, nz = types.shape
    inside = (x < nx) & (y < ny) & (z < nz)
    flat = (np.minimum(x, nx - 1) * ny + np.minimum(y, ny - 1)) * nz + np.minimum(z, nz - 1)
    io = inside & (face[flat] >= 0)
    assert np.array_equal((meta[io] >> 22) & 7, face[flat][io])


@pytest.mark.parametrize("k", ["bad_corner", "bad_interior"])
def test_classify_boundary_faces_rejects_like_reference(golden, k):
    from paper_1611_02445_b200 import boundaries
    gd = golden("faces")
    g = geo_mod.Geometry(gd[f"{k}_types"])
    with pytest.raises(ValueError) as exc:
        boundaries.classify_boundary_faces(g)
    assert str(exc.value) == str(gd[f"{k}_msg"])
    with pytest.raises(ValueError):
        tiling.build_tiling(g)


def test_rejects_bad_faces():
    t = np.ones((8, 8, 8), np.uint8)
    t[0, 0, 0] = 3          # inlet on a corner: three faces
    with pytest.raises(ValueError):
        tiling.build_tiling(geo_mod.Geometry(t))
    t[0, 0, 0] = 9          # unknown tag
    with pytest.raises(ValueError):
        tiling.build_tiling(geo_mod.Geometry(t))


@pytest.mark.parametrize("n,d,p,seed", [(64, 12, 0.5, 1234), (48, 10, 0.2, 7), (96, 20, 0.8, 3),
                                        (20, 8, 0.5, 11), (16, 8, 0.6, 5)])
def test_sphere_pack_on_device_bit_identical(n, d, p, seed):
    """generate_sphere_pack(device=0) (csrc/generate.cu) == the host
    generator (itself bit-identical to the reference), including packs whose
    early passes overshoot the porosity band and restart."""
    from paper_1611_02445_b200 import geometry
    try:
        host = geometry.generate_sphere_pack(n, d, p, seed, inlet_velocity=(0, 0, 0.01))
    except ValueError:
        with pytest.raises(ValueError):
            geometry.generate_sphere_pack(n, d, p, seed, device=0)
        return
    dev = geometry.generate_sphere_pack(n, d, p, seed, inlet_velocity=(0, 0, 0.01), device=0)
    assert np.array_equal(dev.types, host.types)


@pytest.mark.parametrize("shape,levels,seed", [
    ((40, 36, 64), 3, 1), ((33, 47, 29), 2, 5), ((24, 24, 1), 0, 2), ((64, 64, 96), 1, 9),
    ((16, 20, 7), 3, 11)])
def test_vessel_tree_on_device_bit_identical(shape, levels, seed):
    """generate_vessel_tree(device=0) (csrc/generate.cu) == the host builder:
    same lumen discs, walls, inlet and outlet planes."""
    from paper_1611_02445_b200 import geometry
    host = geometry.generate_vessel_tree(shape, levels=levels, seed=seed)
    dev = geometry.generate_vessel_tree(shape, levels=levels, seed=seed, device=0)
    assert np.array_equal(dev.types, host.types)
    assert dev.inlet_velocity == host.inlet_velocity
    assert (host.types == geometry.NodeType.VELOCITY_INLET).any() or shape[2] == 1

"""CPU: geometry generators and TLBM1 I/O vs the reference (golden vectors made
by the reference generators, plus the live reference when mounted)."""

import io

import numpy as np
import pytest

from oracle import dense
from paper_1611_02445_b200 import geometry as g


def test_generators_match_golden(golden):
    gd = golden("tiling")
    mine = {
        "cavity10": g.generate_cavity3d(10),
        "cavity13": g.generate_cavity3d(13),
        "chan_sq": g.generate_channel("square", 9, axis=1, offsets=(1, 2), length=11),
        "chan_ci": g.generate_channel("circle", 10, axis=2, offsets=(3, 1), length=9, ends="io"),
        "pack": g.generate_sphere_pack(22, 8, 0.55, seed=7),
        "pack_x": g.generate_sphere_pack(17, 6, 0.7, seed=3, flow_axis=0),
    }
    for name, geo in mine.items():
        assert np.array_equal(geo.types, gd[f"{name}_types"]), name


def test_sphere_pack_bit_identical_to_reference(reference):
    rg = reference.geometry
    for args in [(32, 8, 0.7, 1), (40, 10, 0.3, 5), (48, 12, 0.5, 1234)]:
        a = rg.generate_sphere_pack(*args, inlet_velocity=(0, 0, 0.01))
        b = g.generate_sphere_pack(*args, inlet_velocity=(0, 0, 0.01))
        assert np.array_equal(a.types, b.types), args
        assert a.porosity() == b.porosity()


def test_channels_and_cavity_match_reference(reference):
    rg = reference.geometry
    assert np.array_equal(rg.generate_cavity3d(7).types, g.generate_cavity3d(7).types)
    for shape in ("square", "circle"):
        for ends in ("wall", "io"):
            for axis in range(3):
                a = rg.generate_channel(shape, 8, axis=axis, offsets=(2, 1), length=6, ends=ends)
                b = g.generate_channel(shape, 8, axis=axis, offsets=(2, 1), length=6, ends=ends)
                assert np.array_equal(a.types, b.types)


def test_generator_errors():
    with pytest.raises(ValueError):
        g.generate_cavity3d(3)
    with pytest.raises(ValueError):
        g.generate_sphere_pack(16, 4, 1.0, seed=1)
    with pytest.raises(ValueError):
        g.generate_channel("hexagon", 8)
    with pytest.raises(ValueError):
        g.generate_channel("square", 8, length=10, ends="periodic")   # not a multiple of 4


def test_box_and_periodic_extensions():
    b = g.generate_box(12)
    assert b.porosity() == 1.0
    assert (b.types[:, :, 0][1:-1, 1:-1] == g.NodeType.VELOCITY_INLET).all()
    c = g.generate_channel("square", 6, axis=0, length=8, ends="periodic")
    assert c.periodic == (True, False, False)
    assert not (c.types == g.NodeType.VELOCITY_INLET).any()


def test_vessel_tree_valid_and_deterministic():
    v = g.generate_vessel_tree((64, 64, 128), levels=3, seed=5)
    w = g.generate_vessel_tree((64, 64, 128), levels=3, seed=5)
    assert v == w
    assert 0.05 < v.porosity() < 0.4
    dense.face_ids(v.types)            # every inlet/outlet node on exactly one face
    assert (v.types == g.NodeType.VELOCITY_INLET).any()
    assert (v.types == g.NodeType.PRESSURE_OUTLET).any()


def test_voxel_roundtrip_and_errors():
    geo = g.generate_cavity3d(9, lid_velocity=(0.02, 0.0, 0.0))
    buf = io.BytesIO()
    g.save_voxels(geo, buf)
    buf.seek(0)
    assert g.load_voxels(buf) == geo
    raw = buf.getvalue()
    for bad in (b"XLBM1" + raw[5:], raw[:30], raw.replace(b"9 9 9", b"9 x 9")):
        with pytest.raises(g.VoxelFormatError):
            g.load_voxels(io.BytesIO(bad))
    one = g.Geometry(np.ones((1, 1, 1), np.uint8))
    buf = io.BytesIO()
    g.save_voxels(one, buf)
    buf.seek(0)
    assert g.load_voxels(buf) == one


def test_voxel_format_matches_reference(reference):
    rg = reference.geometry
    geo = g.generate_sphere_pack(12, 4, 0.6, seed=2)
    a, b = io.BytesIO(), io.BytesIO()
    rg.save_voxels(rg.Geometry(geo.types), a)
    g.save_voxels(g.Geometry(geo.types), b)
    assert a.getvalue() == b.getvalue()

"""CPU: the transaction model (SPEC acceptance 1, 2), the CLI's usage paths
and the output writers (host formatting)."""

import io

import numpy as np
import pytest

from oracle import tiling as ot
from paper_1611_02445_b200 import cli, geometry, layout, output, tiling, txmodel


def test_acceptance1_transaction_arithmetic():
    r = txmodel.count_tile_overheads(layout.LayoutTable.OPTIMIZED, "f64")
    assert (r.tile_read_total, r.tile_read_min) == (344, 304)
    assert abs(r.read_overhead - 0.1316) < 1e-3
    assert r.per_direction_reads["NE"] == 20 and r.per_direction_reads["NW"] == 32
    assert txmodel.count_tile_overheads(layout.LayoutTable.XYZ, "f32").tile_read_total == 288
    assert txmodel.count_tile_overheads(layout.LayoutTable.OPTIMIZED, "f32").tile_read_total == 240
    # the B200 table reaches the minimum when the tile is the request unit
    assert txmodel.count_tile_reads_whole_tile(layout.LayoutTable.B200, "f64") == 304


def test_acceptance2_cavity100_totals():
    g = geometry.generate_cavity3d(100)
    tm, ne = ot.build_tiling(g.types)
    grid = tiling.TileGrid(4, g.shape, (100, 100, 100), tm, ne)
    r = txmodel.geometry_transaction_totals(grid, g, layout.LayoutTable.OPTIMIZED, "f64")
    assert (r.t_n, r.write_segments_min, r.nodetype_read_segments, r.total_min) == \
        (15625, 4750000, 62500, 9562500)
    assert r.tilemap_values_read == 421875


def test_transaction_totals_match_reference(reference):
    rx, rt, rg, rl = reference.txmodel, reference.tiling, reference.geometry, reference.layout
    a = rg.generate_sphere_pack(32, 8, 0.6, seed=5)
    ga = rt.build_tiling(a)
    g = geometry.generate_sphere_pack(32, 8, 0.6, seed=5)
    tm, ne = ot.build_tiling(g.types)
    grid = tiling.TileGrid(4, g.shape, ga.padded_dims, tm, ne)
    for t in ("optimized", "xyz"):
        ra = rx.geometry_transaction_totals(ga, a, rl.LayoutTable(t), "f64")
        rb = txmodel.geometry_transaction_totals(grid, g, layout.LayoutTable(t), "f64")
        for k in ("write_segments_model", "read_segments_model", "total_model", "total_min"):
            assert getattr(ra, k) == getattr(rb, k), k


def test_cli_usage_and_count_tx(capsys):
    assert cli.main(["count-tx", "--precision", "f32", "--layout", "xyz"]) == 0
    assert "total,288" in capsys.readouterr().out
    assert cli.main(["nope"]) == cli.EXIT_USAGE
    with pytest.raises(cli.UsageError):
        cli.parse_geometry("torus:3")


def test_vtk_writer_format_and_determinism():
    rng = np.random.default_rng(0)
    rho = rng.random((3, 2, 4))
    u = rng.random((3, 3, 2, 4))
    a, b = io.StringIO(), io.StringIO()
    output.write_vtk(a, rho, u)
    output.write_vtk(b, rho, u)
    text = a.getvalue()
    assert text == b.getvalue()
    lines = text.splitlines()
    assert lines[0].startswith("# vtk DataFile") and "DIMENSIONS 3 2 4" in lines
    assert "POINT_DATA 24" in lines
    first = lines.index("LOOKUP_TABLE default") + 1
    assert float(lines[first + 1]) == rho[1, 0, 0]          # x fastest
    vec = lines.index("VECTORS velocity double") + 1
    assert [float(v) for v in lines[vec].split()] == list(u[:, 0, 0, 0])


def test_acceptance5_tiling_analytics():
    """SPEC acceptance 5 and the BU_p pin."""
    from paper_1611_02445_b200 import tiling
    assert abs(tiling.overhead_generic(0.83) - 0.2048) < 1e-4
    exact, approx = tiling.overhead_memory(1, 19, 8, 1)
    assert abs(exact - 1.00658) < 1e-5 and approx == 1.0
    assert tiling.overhead_memory(0.5, n_t=0)[0] == 3.0
    assert abs(tiling.bu_propagation_estimate(0, 0) - 0.9212) < 1e-4
    assert tiling.edge_face_plane_residual(2.0, 1.14) == pytest.approx(0.0)
    with pytest.raises(ValueError):
        tiling.bu_propagation_estimate(2.9, 0)


def test_tiling_analytics_match_reference(reference):
    from paper_1611_02445_b200 import tiling
    for ef, ee in ((0.0, 0.0), (1.3, 0.7), (2.5, 2.2)):
        assert tiling.bu_propagation_estimate(ef, ee) == reference.tiling.bu_propagation_estimate(ef, ee)
        assert tiling.edge_face_plane_residual(ef, ee) == reference.tiling.edge_face_plane_residual(ef, ee)


def test_perf_model_matches_reference(reference):
    for kw in ({}, {"n_d": 4}, {"q": 27, "n_d": 8, "n_t": 2}):
        ours, ref = txmodel.PerfModel(**kw), reference.txmodel.PerfModel(**kw)
        assert (ours.m_node(), ours.b_node()) == (ref.m_node(), ref.b_node())


def test_cli_runtime_error_exit_code(capsys):
    """A solver command without a usable configuration fails with exit code 5
    and a one-line message (no traceback)."""
    assert cli.main(["run", "--geometry", "cavity:8", "--precision", "f32", "--arith", "fma"]) == 5
    assert "f64-only" in capsys.readouterr().err


def test_geometry_generators_run_on_the_host_without_a_gpu():
    """workloads / CLI pick the GPU generators only when a GPU is present;
    without one the host builders run (same voxels, tests/test_gpu_tiler.py)."""
    import torch
    from paper_1611_02445_b200 import cli, workloads
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    assert workloads.generator_device() is None
    assert workloads.generator_device(3) == 3
    g = cli.parse_geometry("vessel:24:20:16")
    assert g.shape == (24, 20, 16)
    assert (g.types == 3).any() and (g.types == 4).any()
    with pytest.raises(RuntimeError):
        workloads.vessel_tree((16, 16, 16), device=0)

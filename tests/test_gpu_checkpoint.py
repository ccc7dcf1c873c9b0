"""GPU: checkpoint / resume (Solver.save_checkpoint, solver.resume): a run
interrupted at any iteration and resumed from its checkpoint is
bit-identical to the uninterrupted run."""

import numpy as np
import pytest
import torch

from paper_1611_02445_b200 import cli, geometry, solver

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kw", [{}, {"precision": "f32", "fluid": "quasi-compressible"},
                                {"collision": "mrt"},
                                {"collision": "mrt", "arithmetic": "fma"}])
def test_resume_bit_identical(tmp_path, kw):
    geo = geometry.generate_sphere_pack(24, 6, 0.6, seed=12, inlet_velocity=(0, 0, 0.02))
    cfg = solver.SimulationConfig(u_max_guard=0.0, **kw)
    full = solver.Solver(geo, cfg)
    full.step(31)
    want = full.fields_canonical(device=True)

    a = solver.Solver(geo, cfg)
    a.step(13)                                   # odd iteration: parity 1
    path = tmp_path / "ck.npz"
    a.save_checkpoint(path)
    b = solver.resume(path, geo)                 # config from the checkpoint
    assert b.iteration == 13 and b.parity == 1
    assert b.config.collision == cfg.collision and b.config.arithmetic == cfg.arithmetic
    b.step(18)
    assert torch.equal(b.fields_canonical(device=True), want)


def test_resume_rejects_other_geometry(tmp_path):
    g1 = geometry.generate_cavity3d(12)
    s = solver.Solver(g1)
    s.step(2)
    s.save_checkpoint(tmp_path / "ck.npz")
    g2 = geometry.generate_cavity3d(12, lid_velocity=(0.04, 0.0, 0.0))
    with pytest.raises(ValueError, match="another geometry"):
        solver.resume(tmp_path / "ck.npz", g2)
    with pytest.raises(ValueError, match="do not fit"):
        solver.Solver(g1, solver.SimulationConfig(precision="f32")).load_checkpoint(
            tmp_path / "ck.npz")


def test_cli_run_checkpoint_resume(tmp_path, capsys):
    ck1, ck2 = tmp_path / "a.npz", tmp_path / "b.npz"
    assert cli.main(["run", "--geometry", "cavity:16", "--iters", "70", "--graph", "on",
                     "--checkpoint", str(ck1)]) == 0
    assert cli.main(["run", "--geometry", "cavity:16", "--iters", "30", "--resume", str(ck1),
                     "--checkpoint", str(ck2)]) == 0
    s = solver.Solver(geometry.generate_cavity3d(16))
    s.run(100)
    with np.load(ck2) as z:
        assert int(z["iteration"]) == 100
        assert np.array_equal(z["f"], s.fields_canonical())

"""GPU: the CUDA-graph run path (Solver.step(graph=True)): blocks of
GRAPH_STEPS step launches captured once and replayed, the status slot taken
from a device iteration counter (tlbm_step_args.iter_counter) instead of a
per-launch host pointer.  Results must be bit-identical to launching the
same steps one by one, and divergence / guard reporting must keep the exact
iteration."""

import warnings

import numpy as np
import pytest
import torch

from oracle import dense
from paper_1611_02445_b200 import collision, geometry, solver
from test_gpu_step import MODELS, compare, make_solver, oracle_run

pytestmark = pytest.mark.gpu
K = solver.GRAPH_STEPS


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("coll", ["lbgk", "mrt"])
def test_graph_equals_launches(prec, coll):
    # LBGK on a sphere pack with inlet/outlet; MRT (default rates, which a
    # 28^3 Zou-He pack drives unstable) on a periodic channel
    geo = (geometry.generate_sphere_pack(28, 8, 0.6, seed=4, inlet_velocity=(0, 0, 0.02))
           if coll == "lbgk" else
           geometry.generate_channel("square", 18, axis=2, offsets=(1, 2), length=28,
                                     ends="periodic"))
    runs = []
    for mode in ("launch", "graph", "mixed"):
        cfg = solver.SimulationConfig(collision=coll, precision=prec, u_max_guard=0.0)
        s = solver.Solver(geo, cfg)
        s.init_equilibrium(1.0, (0.0, 0.0, 0.01))
        n = 3 * K + 7
        if mode == "launch":
            s.step(n)
        elif mode == "graph":
            s.step(n, graph=True)
        else:                        # odd start parity, then graph blocks, then launches
            s.step(5)
            s.step(2 * K + 1, graph=True)
            s.step(n - 5 - 2 * K - 1, graph=True)
        assert s.iteration == n
        runs.append(s.fields_canonical(device=True))
    assert torch.equal(runs[0], runs[1]) and torch.equal(runs[0], runs[2])


def test_graph_cavity_matches_oracle(c_oracle):
    geo = geometry.generate_cavity3d(24)
    m = MODELS["inc"]
    f0 = dense.init_equilibrium(geo.shape, m, np.float64)
    s = make_solver(geo, m, np.float64)
    s.run(5 * K, graph=True)
    compare(s, oracle_run(c_oracle, geo, m, np.float64, f0, 5 * K), np.float64)


def test_graph_divergence_reports_iteration():
    geo = geometry.Geometry(np.ones((8, 8, 8), np.uint8), periodic=(True, True, True))
    s = make_solver(geo, MODELS["inc"], np.float64)
    s.step(K + 3, graph=True)
    f = s.fields_canonical()
    f[:, 0, 5] = np.nan
    s.store.fill_canonical(s.parity, f)
    with pytest.raises(collision.DivergenceError) as ei:
        s.step(2 * K, graph=True)
    assert ei.value.iteration == K + 3


def test_graph_guard_iterations_wrap_the_ring():
    """Guard trips are recorded per iteration across status-ring wrap-around
    (STATUS_RING is a multiple of GRAPH_STEPS; start at an offset)."""
    geo = geometry.Geometry(np.ones((8, 8, 8), np.uint8), periodic=(True, True, True))
    s = make_solver(geo, MODELS["inc"], np.float64, guard=0.05)
    s.init_equilibrium(1.0, (0.08, 0.0, 0.0))
    s.iteration = s._checked = solver.STATUS_RING - 10
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s.step(2 * K, graph=True)
    assert s.guard_iterations == list(range(solver.STATUS_RING - 10,
                                            solver.STATUS_RING - 10 + 2 * K))

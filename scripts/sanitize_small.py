"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / initcheck) on the GPU box."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_02445_b200 import _native as nat  # noqa: E402
from paper_1611_02445_b200 import collision, geometry, slabs, solver  # noqa: E402

geo = geometry.generate_sphere_pack(20, 6, 0.6, seed=3, inlet_velocity=(0, 0, 0.02))
assert (geometry.generate_sphere_pack(20, 6, 0.6, seed=3, inlet_velocity=(0, 0, 0.02),
                                      device=0).types == geo.types).all()
for prec in ("f64", "f32"):
    for fluid in ("incompressible", "quasi-compressible"):
        s = solver.Solver(geo, solver.SimulationConfig(precision=prec, fluid=fluid))
        s.step(3)
        s.step(1, variant=nat.PROPAGATION_ONLY)
        s.step(1, variant=nat.READ_WRITE_ONLY)
        s.macroscopic()
        s.fields_canonical()
for coll in ("lbgk", "mrt"):
    for prec in ("f64", "f32"):
        s = solver.Solver(geo, solver.SimulationConfig(collision=coll, precision=prec))
        s.step(2)
        s = solver.Solver(geo, solver.SimulationConfig(collision=coll, precision=prec), index64=True)
        s.step(2)
    s = solver.Solver(geo, solver.SimulationConfig(collision=coll, arithmetic="fma"))
    s.step(2)
chan = geometry.generate_channel("square", 12, axis=2, length=24, ends="periodic")
for fused in (False, True):
    for storage, trav in (("blocks", "tile"), ("compact", "tile"), ("compact", "nodes")):
        vs = slabs.VirtualSlabs(chan, 3, solver.SimulationConfig(storage=storage), fused=fused,
                                traversal=trav)
        vs.step(3)
for prec in ("f64", "f32"):
    for trav in ("tile", "nodes"):        # tile- and node-parallel compact steps
        s = solver.Solver(geo, solver.SimulationConfig(precision=prec, storage="compact"),
                          traversal=trav)
        s.step(2)
        s.step(1, variant=nat.PROPAGATION_ONLY)
        s.step(1, variant=nat.READ_WRITE_ONLY)
        s.macroscopic()
        s.fields_canonical()
        s = solver.Solver(geo, solver.SimulationConfig(precision=prec, storage="compact",
                                                       collision="mrt"), traversal=trav)
        s.step(2)
for trav in ("tile", "nodes"):
    s = solver.Solver(geo, solver.SimulationConfig(collision="mrt", storage="compact",
                                                   arithmetic="fma"), traversal=trav)
    s.step(2)
solver.GRAPH_STEPS = 4
s = solver.Solver(geo, solver.SimulationConfig())
s.step(9, graph=True)
f = np.random.default_rng(0).random((19, 10))
collision.collide_lbgk("incompressible", f, 0.7)
print("sanitize run ok")

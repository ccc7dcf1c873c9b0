import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1611_02445_b200 import geometry, solver
geo = geometry.generate_sphere_pack(30, 8, 0.55, seed=21, inlet_velocity=(0, 0, 0.02))
prec, coll = sys.argv[1], sys.argv[2]
cfg = solver.SimulationConfig(collision=coll, tau=0.6, u_max_guard=0.0, precision=prec)
s = solver.Solver(geo, cfg, index64=True)
s.step(3)
print(prec, coll, "ok")

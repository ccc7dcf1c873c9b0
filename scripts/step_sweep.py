"""Time the step kernel variants (full / propagation-only / read-write-only)
on a workload; prints one JSON line per (variant).  Used for tuning runs on
the GPU box: TLBM_LIB selects an alternative build of libtlbm.so."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_02445_b200 import _native as nat  # noqa: E402
from paper_1611_02445_b200 import workloads  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=256)
p.add_argument("--precision", default="f64")
p.add_argument("--table", default=None, help="layout table (default: b200, xyz if compact)")
p.add_argument("--steps", type=int, default=100)
p.add_argument("--variants", default="full,prop,rw")
p.add_argument("--geometry", default="channel",
               help="channel | channel_z | duct_z | cavity | pack | vessel")
p.add_argument("--length", type=int, default=None, help="channel_z length along z")
p.add_argument("--dims", default="512,512,1024", help="vessel dims nx,ny,nz")
p.add_argument("--no-perturb", action="store_true",
               help="uniform equilibrium start (no (t_n, 64) init temporaries; big domains)")
p.add_argument("--porosity", type=float, default=0.5)
p.add_argument("--index64", action="store_true", help="force 64-bit addressing")
p.add_argument("--arith", default="reference", choices=["reference", "fma"])
p.add_argument("--graph", action="store_true", help="replay captured CUDA graphs of steps")
p.add_argument("--storage", default="blocks", choices=["blocks", "compact"])
p.add_argument("--traversal", default="auto", help="auto | tile | <rows per band>")
p.add_argument("--l2-fetch", type=int, default=-1,
               help="cudaLimitMaxL2FetchGranularity in bytes (0..128; -1 leaves the default)")
a = p.parse_args()
traversal = int(a.traversal) if a.traversal.isdigit() else a.traversal
if a.geometry == "channel":
    geo = workloads.channel(a.n)
elif a.geometry == "channel_z":
    geo = workloads.channel_z(a.n, a.length)
elif a.geometry == "duct_z":        # walled square duct along z (no periodic wrap)
    from paper_1611_02445_b200 import geometry as _g
    geo = _g.generate_channel("square", a.n, axis=2, length=a.length or a.n, ends="wall")
elif a.geometry == "vessel":        # tortuous vessel tree (BASELINE configs 4 and 5)
    geo = workloads.vessel_tree(tuple(int(v) for v in a.dims.split(",")))
elif a.geometry == "cavity":
    geo = workloads.cavity(a.n)
else:
    geo = workloads.sphere_pack(a.porosity, n=a.n)
s = workloads.make_solver(geo, precision=a.precision, table=a.table, u0=(0.04, 0, 0),
                          index64=a.index64, arithmetic=a.arith, perturb=not a.no_perturb,
                          storage=a.storage,
                          traversal=traversal)
if a.no_perturb:
    s.init_equilibrium(1.0, (0.0, 0.0, 0.04) if a.geometry == "channel_z" else (0.04, 0.0, 0.0))
from paper_1611_02445_b200.solver import GRAPH_STEPS as solver_graph_steps  # noqa: E402
l2_fetch = None
if a.l2_fetch >= 0:
    nat.call("tlbm_set_l2_fetch_granularity", a.l2_fetch)
    _v = nat.ctypes.c_int()
    nat.call("tlbm_get_l2_fetch_granularity", nat.ctypes.byref(_v))
    l2_fetch = _v.value
vmap = {"full": nat.FULL, "prop": nat.PROPAGATION_ONLY, "rw": nat.READ_WRITE_ONLY,
        "mrt": nat.FULL}
n_d = 8 if a.precision == "f64" else 4
solvers = {"lbgk": s}
for v in a.variants.split(","):
    if v == "mrt" and "mrt" not in solvers:
        from paper_1611_02445_b200.solver import SimulationConfig, Solver
        cfg = SimulationConfig(collision="mrt", tau=workloads.TAU, precision=a.precision,
                               table=a.table, u_max_guard=0.0, arithmetic=a.arith,
                               storage=a.storage)
        del solvers["lbgk"], s
        torch.cuda.empty_cache()
        s = solvers["mrt"] = Solver(geo, cfg, index64=a.index64, traversal=traversal)
    s.step(solver_graph_steps if a.graph else 5, variant=vmap[v], check=False, graph=a.graph)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step(a.steps, variant=vmap[v], check=False, graph=a.graph)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    mlups = s.n_fn / (ms / 1e3) / 1e6
    gbs = s.n_fn * 2 * 19 * n_d / (ms / 1e3) / 1e9
    print(json.dumps({"lib": os.path.basename(nat.LIB_PATH), "index64": a.index64,
                      "arith": a.arith, "graph": a.graph, "l2_fetch": l2_fetch,
                      "storage": a.storage, "ordered": s.order is not None,
                      "geometry": a.geometry, "n": a.n, "dims": list(geo.shape),
                      "field_gb": round(s.store.flat.numel() * n_d / 1e9, 2),
                      "precision": a.precision, "table": a.table, "variant": v,
                      "ms": round(ms, 4), "mlups": round(mlups, 1), "gbs": round(gbs, 1),
                      "frac": round(gbs / 6533.5, 4), "n_fn": s.n_fn, "t_n": s.t_n}), flush=True)

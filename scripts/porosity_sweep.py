"""BASELINE config 3/4 sweep: sphere packs 256^3 (d = 40, seed 1234) over
porosity 0.2..1.0 and the 512x512x1024 vessel tree, fp64 and fp32.

For every case prints one JSON line: t_n, n_fn, porosity, eta_t, ms/step
(CUDA events over --steps launches after --warmup), MLUPS, and bandwidth
utilisation BU = MLUPS * 1e6 * B_node / hbm_gbs (B_node = 304 / 152 B,
PAPER.md:947; hbm_gbs from MEASURED_PEAKS.json) -- the paper's Table 5/6
quantities on one B200.

    python scripts/porosity_sweep.py [--precisions f64,f32] [--porosities ...]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1611_02445_b200 import workloads  # noqa: E402
from paper_1611_02445_b200.solver import SimulationConfig, Solver  # noqa: E402


def hbm_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def time_case(name, geo, precision, steps, warmup, table, storage="blocks"):
    t0 = time.perf_counter()
    # "nodes": compact storage, node-parallel step; "compact": compact
    # storage, tile-parallel step; "auto": what the solver picks
    cfg = SimulationConfig(tau=workloads.TAU, precision=precision, table=table,
                           u_max_guard=0.0, storage="compact" if storage == "nodes" else storage)
    s = Solver(geo, cfg, traversal="nodes" if storage == "nodes"
               else ("tile" if storage == "compact" else "auto"))
    setup = time.perf_counter() - t0
    s.step(warmup, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step(steps, check=False)
    e1.record()
    torch.cuda.synchronize()
    s.check()
    ms = e0.elapsed_time(e1) / steps
    b_node = 304 if precision == "f64" else 152
    mlups = s.n_fn / (ms / 1e3) / 1e6
    rec = {"case": name, "precision": precision, "table": s.config.table.value,
           "storage": storage, "storage_used": s.config.storage,
           "traversal_used": "nodes" if s.nodes is not None else "tile",
           "dims": list(geo.shape),
           "porosity": geo.porosity(), "t_n": s.t_n, "n_fn": s.n_fn,
           "eta_t": s.n_fn / (64 * s.t_n), "ms_per_step": ms, "mlups": mlups,
           "bu": mlups * 1e6 * b_node / (hbm_gbs() * 1e9), "setup_s": setup, "steps": steps}
    del s
    torch.cuda.empty_cache()
    return rec


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--precisions", default="f64,f32")
    p.add_argument("--porosities", default="0.2,0.3,0.4,0.5,0.6,0.7,0.8,0.9,1.0")
    p.add_argument("--n", type=int, default=256)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--table", default=None, help="default: b200 (blocks), xyz (compact)")
    p.add_argument("--vessel", action="store_true")
    p.add_argument("--cavity", action="store_true")
    p.add_argument("--l2-fetch", type=int, default=-1)
    p.add_argument("--storages", default="blocks", help="comma list of blocks,compact,nodes,auto")
    a = p.parse_args()
    if a.l2_fetch >= 0:
        from paper_1611_02445_b200 import _native as nat
        nat.require_cuda()
        nat.call("tlbm_set_l2_fetch_granularity", a.l2_fetch)
        v = nat.c_int(0)
        nat.call("tlbm_get_l2_fetch_granularity", nat.ctypes.byref(v))
        print(json.dumps({"l2_fetch_granularity": v.value}), flush=True)
    cases = []
    for por in (float(v) for v in a.porosities.split(",") if v):
        t0 = time.perf_counter()
        geo = workloads.sphere_pack(por, n=a.n)
        cases.append((f"spheres_p{por:.1f}", geo, time.perf_counter() - t0))
    if a.vessel:
        t0 = time.perf_counter()
        cases.append(("vessel_512x512x1024", workloads.vessel_tree(), time.perf_counter() - t0))
    if a.cavity:
        cases.append(("cavity64", workloads.cavity(64), 0.0))
    for name, geo, gen_s in cases:
        for storage in a.storages.split(","):
            for prec in a.precisions.split(","):
                rec = time_case(name, geo, prec, a.steps, a.warmup, a.table, storage)
                rec["geometry_s"] = gen_s
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

"""Where the end-to-end setup time of the bench workload goes (GPU box):
host-clock times (synchronised) of the pieces of DistributedSlabRunner(
geometry) at N = 1 -- tags H2D (pageable vs pinned), device tiler, solver
(allocation + initial equilibrium) -- and of the rho/u readout.

    python scripts/e2e_phases.py [--edge 256] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1611_02445_b200 import slabs, solver, tiling, workloads  # noqa: E402


def clock(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edge", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    geo = workloads.channel_z(a.edge)
    tags = torch.empty(geo.shape, dtype=torch.uint8, pin_memory=True)
    tags.numpy()[...] = geo.types
    pinned_geo = type(geo)(tags.numpy(), geo.inlet_velocity, geo.outlet_density,
                           periodic=geo.periodic)
    cfg = solver.SimulationConfig(tau=0.6)
    for rep in range(a.reps):
        rec = {"rep": rep}
        _, rec["h2d_pageable_ms"] = clock(lambda: torch.from_numpy(geo.types).cuda())
        _, rec["h2d_pinned_ms"] = clock(lambda: torch.from_numpy(pinned_geo.types).cuda())
        tl, rec["device_tiling_ms"] = clock(lambda: tiling.DeviceTiling(pinned_geo))
        s, rec["solver_ms"] = clock(lambda: solver.Solver(pinned_geo, cfg, tiling=tl,
                                                          initial=(1.0, (0, 0, 0.02))))
        _, rec["init_equilibrium_ms"] = clock(lambda: s.init_equilibrium(1.0, (0, 0, 0.02)))
        del s, tl
        run, rec["runner_ms"] = clock(lambda: slabs.DistributedSlabRunner(
            pinned_geo, 1, 0, cfg, initial=(1.0, (0, 0, 0.02))))
        s = run.slab.solver
        rho = torch.empty((s.t_n, 64), dtype=torch.float64, pin_memory=True)
        u = torch.empty((3, s.t_n, 64), dtype=torch.float64, pin_memory=True)
        (rd, ud, _), rec["macroscopic_ms"] = clock(lambda: s.macroscopic(device=True))
        _, rec["d2h_rho_u_ms"] = clock(lambda: (rho.copy_(rd, non_blocking=True),
                                                u.copy_(ud, non_blocking=True)))
        rec["d2h_gbs"] = (rho.numel() + u.numel()) * 8 / rec["d2h_rho_u_ms"] / 1e6
        del run, s, rd, ud
        print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v)
                          for k, v in rec.items()}), flush=True)


if __name__ == "__main__":
    main()

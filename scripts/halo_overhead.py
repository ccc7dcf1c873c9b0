"""Cost of the multi-GPU code path, measured on one GPU.

The weak-scaling bench workload for N ranks (256 x 256 x 256N channel,
periodic z) is run (a) as one domain and (b) as N z slabs one after another
on the same GPU (slabs.VirtualSlabs): interior launch, then the boundary
layers with the halo stored into the neighbour slab's ghost tiles -- the
fused-halo kernels of the IPC path with device pointers in place of NVLink
peer mappings (fused), or pack -> device copy -> unpack (the NCCL path's
data flow).  (b) / (a) - 1 is the per-step overhead of the decomposition
itself (split launches, halo stores, ghost layers) -- everything the N-GPU
step adds except the NVLink transfer latency and the neighbour wait, which
one GPU cannot show.

    python scripts/halo_overhead.py [--ranks 2,4,8] [--precision f64] [--steps 20]
        [--geometry channel|pack --porosity 0.2 --storage blocks|compact|auto]

``--geometry pack``: the 256^3 sphere pack of BASELINE config 3 cut into N
slabs (the same domain, so per-slab work shrinks with N), with the storage
and step that ``--storage`` selects (auto: compact + node-parallel below
eta_t 0.93).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1611_02445_b200 import slabs, workloads  # noqa: E402
from paper_1611_02445_b200.solver import SimulationConfig, Solver  # noqa: E402


def timed(step, steps):
    step(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step(steps)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ranks", default="2,4,8")
    p.add_argument("--precision", default="f64")
    p.add_argument("--edge", type=int, default=256)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--geometry", default="channel", choices=["channel", "pack"])
    p.add_argument("--porosity", type=float, default=0.2)
    p.add_argument("--storage", default="blocks")
    a = p.parse_args()
    cfg = SimulationConfig(tau=workloads.TAU, precision=a.precision, u_max_guard=0.0,
                           storage=a.storage)
    pack = workloads.sphere_pack(a.porosity, n=a.edge) if a.geometry == "pack" else None
    for n in (int(v) for v in a.ranks.split(",")):
        geo = pack if pack is not None else workloads.channel_z(a.edge, a.edge * n)
        s = Solver(geo, cfg)
        s.init_equilibrium(1.0, (0.0, 0.0, 0.04))
        t_one = timed(lambda k: s.step(k, check=False), a.steps)
        n_fn = s.n_fn
        del s
        torch.cuda.empty_cache()
        rec = {"ranks": n, "precision": a.precision, "geometry": a.geometry,
               "storage": a.storage, "dims": list(geo.shape), "n_fn": n_fn,
               "ms_one_domain": t_one}
        for fused in (True, False):
            vs = slabs.VirtualSlabs(geo, n, cfg, fused=fused)
            rec["nodes_step"] = all(sl.solver.nodes is not None for sl in vs.slabs)
            for sl in vs.slabs:
                sl.solver.init_equilibrium(1.0, (0.0, 0.0, 0.04))
            t = timed(vs.step, a.steps)
            key = "fused" if fused else "pack_copy_unpack"
            rec[f"ms_slabs_{key}"] = t
            rec[f"overhead_{key}"] = t / t_one - 1.0
            del vs
            torch.cuda.empty_cache()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

"""Why the bench line's fp64 step (0.787 ms) is ~2.5% slower than the
step_sweep ladder's (0.767 ms) on the same kernel: time 200 steps of the
256^3 channel as (a) step_sweep builds it (Solver, u0 = 0.04 along x),
(b) the same with the bench's u0 = 0.02 along z, (c) bench's SlabWorkload
at N = 1, (d) (c) with bench's NVML clock sampler running."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1611_02445_b200 import slabs, workloads  # noqa: E402


def timed(step, n=200):
    step(5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step(n)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


geo = workloads.channel_z(256)
for rep in range(2):
    out = {}
    s = workloads.make_solver(geo, "f64")
    out["a_solver_u0x"] = timed(lambda n: s.step(n, check=False))
    del s
    torch.cuda.empty_cache()
    s = workloads.make_solver(geo, "f64", u0=(0.0, 0.0, 0.02))
    out["b_solver_u0z"] = timed(lambda n: s.step(n, check=False))
    del s
    torch.cuda.empty_cache()
    r = slabs.SlabWorkload(geo, 1, 0, transport="ipc")
    out["c_slab"] = timed(lambda n: r.step(n, check=False))
    with bench.ClockSampler(0):
        out["d_slab_sampler"] = timed(lambda n: r.step(n, check=False))
    with bench.ClockSampler(0):
        s2 = r.slab.solver
        out["e_slab_solver_step_sampler"] = timed(lambda n: s2.step(n, check=False))
    del r, s2
    torch.cuda.empty_cache()
    print(json.dumps({k: round(v, 4) for k, v in out.items()}), flush=True)

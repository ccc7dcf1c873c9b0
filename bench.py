"""Benchmark of the tiled D3Q19 LBGK step on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N = 1 workload: BASELINE config 2 -- dense square channel 256^3, bounce-back
ring, periodic along its axis z, LBGK incompressible, fp64, tau = 0.6, started from a
perturbed equilibrium (paper_1611_02445_b200/workloads.py).  One "step" = one
launch of the fused collide+propagate kernel over all 262,144 tiles.  The
field (2 x 2.55 GB) is far larger than L2 (126 MB), so no flush is needed.

N > 1 (torchrun, one rank per GPU): weak scaling -- every rank owns a
256^3 z-slab of a 256 x 256 x 256N channel periodic in z; the boundary tile
layers' outgoing z planes are exchanged every step over NCCL, overlapped with
the interior-tile launch (paper_1611_02445_b200/slabs.py).

Reported (one JSON line on rank 0):
  value      MLUPS over all ranks (non-solid node updates / s / 1e6), device
             time from CUDA events on the launching stream, max over ranks
  roofline   algorithmic bytes per launch = n_fn x 2 x 19 x 8 B (txmodel
             b_node) / average launch time, vs MEASURED_PEAKS.json hbm_gbs;
             traffic = ncu dram bytes per launch (profiles/roofline_traffic.json)
  e2e        the same metric through the public API from host data: geometry
             upload, device tiling, init, K steps each followed by an async
             D2H of the step's status word, final rho/u readout to the host
  cpu_baseline  the C oracle (oracle/tlbm_oracle.c, OpenMP on all host cores)
             on a bounded sample of the same workload (rank 0, N = 1)
  porosity   the "vs porosity" part of the metric (rank 0, N = 1): MLUPS and
             BU = MLUPS x 304 B / peak on the 256^3 sphere packs (BASELINE
             config 3; d = 40, seed 1234) at porosity 0.2 / 0.5 / 0.9 / 1.0,
             for the paper's block storage and for storage="auto"
  --impl reference  times that same CPU oracle as the reference arm
"""

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "D3Q19 fp64 MFLUPS and % of peak HBM GB/s vs porosity at 1/2/4/8 B200"
UNIT = "MFLUPS"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--precision", default="f64", choices=["f64", "f32"])
    p.add_argument("--edge", type=int, default=256, help="channel edge in nodes")
    p.add_argument("--table", default="b200")
    p.add_argument("--arith", default="reference", choices=["reference", "fma"],
                   help="collision arithmetic: reference = bit-exact unfused order, "
                        "fma = fused multiply-adds (parity within tolerance)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-sweep", action="store_true", help="skip the porosity block")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--transport", default="ipc", choices=["ipc", "nccl", "gloo"],
                   help="N>1 halo: ipc = fused peer stores from the step kernel (default), "
                        "nccl = pack + NCCL send/recv + unpack, gloo = host-staged (tests)")
    return p.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, index, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover - depends on the box
            self.err = str(exc)

    def _run(self):
        n = self.nvml
        names = {
            "hw_slowdown": getattr(n, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(n, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(n, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(n, "nvmlClocksEventReasonHwPowerBrakeSlowdown",
                                               0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM))
                r = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self.t.join()

    def report(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def traffic_from_profiles(key):
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    return d.get(key)


# ---------------------------------------------------------------- CPU oracle
def cpu_oracle_mlups(precision, n, seconds, threads=0):
    """C oracle (OpenMP, `threads` = all available) on a bounded sample of the
    channel workload: the same 256 x 256 cross-section, 32 nodes along the
    periodic axis (per-node work is identical along the channel)."""
    from oracle import c_oracle, dense
    from paper_1611_02445_b200 import workloads
    dt = np.float64 if precision == "f64" else np.float32
    length = 32
    geo = workloads.channel_z(n, length=length)
    f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.04))
    cores = threads or len(os.sched_getaffinity(0))
    o = c_oracle.DenseOracle(geo.types, "incompressible", workloads.TAU, periodic=geo.periodic,
                             f0=f0, dtype=dt, nthreads=cores)
    n_fn = geo.nonsolid_count()
    o.run(1)                                     # warm-up (page faults, threads)
    steps, t0 = 0, time.perf_counter()
    while True:
        o.run(1)
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds or steps >= 200:
            break
    return {"value": n_fn * steps / el / 1e6, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"C oracle (oracle/tlbm_oracle.c, OpenMP x{cores}) on the channel "
                      f"{n}x{n}x{length} slab (periodic z), {precision}, {steps} steps "
                      f"in {el:.1f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    t_all = []
    from oracle import c_oracle, dense
    from paper_1611_02445_b200 import workloads
    dt = np.float64 if args.precision == "f64" else np.float32
    length = 32
    geo = workloads.channel_z(args.edge, length=length)
    f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.04))
    cores = len(os.sched_getaffinity(0))
    o = c_oracle.DenseOracle(geo.types, "incompressible", workloads.TAU, periodic=geo.periodic,
                             f0=f0, dtype=dt, nthreads=cores)
    n_fn = geo.nonsolid_count()
    for _ in range(args.warmup):
        o.run(1)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.run(1)
        t_all.append(time.perf_counter() - t0)
    total = sum(t_all)
    value = n_fn * args.steps / total / 1e6
    sample = (f"C oracle port (oracle/tlbm_oracle.c, OpenMP x{cores}): each step = one full "
              f"step of the channel {args.edge}x{args.edge}x{length} slab (periodic z), "
              f"{args.precision}; the reference has no step of its own (SURVEY 0.2)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": f"channel{args.edge}_periodic_{args.precision}",
                       "sample_nodes": n_fn},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def e2e_run(args, torch, geo_host, world, rank, dist):
    """Public API end to end from host data, on every rank:
    DistributedSlabRunner(geometry) [slab cut, H2D of the local tags, device
    tiler + metadata, init, initial ghost exchange], K x step() each followed
    by an async D2H of that step's status word to pinned memory, and the final
    rho/u readout of the owned tiles into pinned host buffers (allocated once,
    outside the timed region, like the status buffer).  Time = max over ranks;
    phase times (host clock, a sync at each phase end) reported beside it."""
    from paper_1611_02445_b200 import slabs
    from paper_1611_02445_b200 import solver as sv
    cfg = sv.SimulationConfig(tau=0.6, precision=args.precision, table=args.table,
                              arithmetic=args.arith)
    dt = torch.float64 if args.precision == "f64" else torch.float32
    plan = slabs.SlabPlan(geo_host, world)
    r = plan.ranges[rank]
    t_own = _tiles_in(geo_host.types[:, :, r.z0:r.z1])
    pinned = torch.empty(max(args.steps, args.warmup), dtype=torch.int32, pin_memory=True)
    rho = torch.empty((t_own, 64), dtype=dt, pin_memory=True)
    u = torch.empty((3, t_own, 64), dtype=dt, pin_memory=True)
    # one untimed pass of the whole e2e path with `warmup` steps first: a
    # serving process has its CUDA context, modules and caching-allocator
    # blocks already; the timed pass then measures the per-job work, not
    # first-use cudaMalloc of the 5 GB field store
    _e2e_pass(args, torch, geo_host, world, rank, dist, cfg, pinned, rho, u, args.warmup)
    el, t0, t1, t2, t3, n_fn, h2d, d2h = _e2e_pass(args, torch, geo_host, world, rank, dist, cfg,
                                                   pinned, rho, u, args.steps)
    if dist is not None:
        v = torch.tensor([el, n_fn, h2d, d2h], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        mx = v.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(v)
        el, n_fn, h2d, d2h = float(mx[0]), int(v[1]), float(v[2]), float(v[3])
    return {"value": n_fn * args.steps / el / 1e6, "unit": UNIT,
            "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
            "seconds": el,
            "phases": {"setup_s": t1 - t0, "steps_s": t2 - t1, "readout_s": t3 - t2},
            "what": "DistributedSlabRunner(geometry) + init + K x step() with per-step async "
                    "D2H of the status word + final owned rho/u readout to pinned host "
                    "memory; max over ranks; after one untimed warm-up pass of the same path"}


def _e2e_pass(args, torch, geo_host, world, rank, dist, cfg, pinned, rho, u, steps):
    from paper_1611_02445_b200 import slabs
    from paper_1611_02445_b200 import solver as sv
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run = slabs.DistributedSlabRunner(geo_host, world, rank, cfg,
                                      transport=getattr(args, "transport_used", args.transport))
    s = run.slab.solver
    s.init_equilibrium(1.0, (0.0, 0.0, 0.04))
    run.exchange_current()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for i in range(steps):
        run.step(1)
        slot = (s.iteration - 1) % sv.STATUS_RING
        pinned[i:i + 1].copy_(s.status[slot:slot + 1], non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rho_d, u_d, _ = s.macroscopic(device=True)
    b, e = run.slab.own
    rho.copy_(rho_d[b:e], non_blocking=True)
    u.copy_(u_d[:, b:e], non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    el = t3 - t0
    if np.any(pinned[:steps].numpy() & 1):
        raise RuntimeError("e2e run diverged")
    n_fn = run.n_fn_owned
    if run.ipc is not None:
        run.ipc.check()
        run.ipc.close()
    h2d = run.slab.local_geometry.types.nbytes
    d2h = 4 * steps + rho.numel() * rho.element_size() + u.numel() * u.element_size()
    del run, s, rho_d, u_d
    return el, t0, t1, t2, t3, n_fn, h2d, d2h


def porosity_block(args, torch, porosities=(0.2, 0.5, 0.9, 1.0), steps=20):
    """BASELINE config 3 at four porosities, CUDA events over `steps`
    launches after 3 warm-up launches, for both the paper's block storage
    and storage="auto" (compact fp64 storage below tile utilisation 0.88)."""
    from paper_1611_02445_b200 import workloads
    from paper_1611_02445_b200.solver import SimulationConfig, Solver
    peak, _ = peaks()
    n_d = 8 if args.precision == "f64" else 4
    out = {"workload": "sphere pack 256^3, d=40, seed 1234 (porosity 1.0: all-fluid box)",
           "precision": args.precision, "porosity": list(porosities), "eta_t": [],
           "mlups_blocks": [], "bu_blocks": [], "mlups_auto": [], "bu_auto": [],
           "storage_auto": []}
    for por in porosities:
        geo = workloads.sphere_pack(por, n=args.edge)
        for storage in ("blocks", "auto"):
            cfg = SimulationConfig(tau=workloads.TAU, precision=args.precision,
                                   u_max_guard=0.0, storage=storage)
            s = Solver(geo, cfg)
            s.step(3, check=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.step(steps, check=False)
            e1.record()
            torch.cuda.synchronize()
            s.check()
            mlups = s.n_fn * steps / (e0.elapsed_time(e1) / 1e3) / 1e6
            out[f"mlups_{storage}"].append(round(mlups, 1))
            out[f"bu_{storage}"].append(round(mlups * 1e6 * 2 * 19 * n_d / (peak * 1e9), 4))
            if storage == "auto":
                out["storage_auto"].append(s.config.storage)
            else:
                out["eta_t"].append(round(s.n_fn / (64 * s.t_n), 4))
            del s
            torch.cuda.empty_cache()
    return out


def _tiles_in(types):
    """Non-empty 4^3 tiles of a voxel block (sizes the pinned result buffers)."""
    nx, ny, nz = types.shape
    pad = np.zeros(tuple(-(-n // 4) * 4 for n in types.shape), dtype=bool)
    pad[:nx, :ny, :nz] = types != 0
    m = pad.reshape(pad.shape[0] // 4, 4, pad.shape[1] // 4, 4, pad.shape[2] // 4, 4)
    return int(m.any(axis=(1, 3, 5)).sum())


def run_b200(args):
    import torch
    from paper_1611_02445_b200 import _native as nat
    from paper_1611_02445_b200 import txmodel, workloads

    rank, world, local = dist_env()
    shared = torch.cuda.device_count() < world      # test mode: ranks share one GPU
    if shared and args.transport == "nccl":
        raise SystemExit("NCCL needs one GPU per rank; use --transport ipc|gloo to share one")
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    backend = "gloo" if (shared or args.transport == "gloo") else "nccl"
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_1611_02445_b200 import slabs
    transport = args.transport
    try:
        runner = slabs.SlabChannel(args.edge, world, rank, precision=args.precision,
                                   table=args.table, transport=transport, arithmetic=args.arith)
    except RuntimeError as exc:
        if transport != "ipc":
            raise
        print(f"[bench] ipc halo unavailable ({exc}); falling back to nccl", file=sys.stderr)
        transport = "nccl" if backend == "nccl" else "gloo"
        runner = slabs.SlabChannel(args.edge, world, rank, precision=args.precision,
                                   table=args.table, transport=transport, arithmetic=args.arith)
    args.transport_used = transport
    n_fn_rank = runner.n_fn_owned
    step_fn = runner.step
    sync_all = runner.barrier

    for _ in range(args.warmup):
        step_fn(1)
    torch.cuda.synchronize()
    sync_all()

    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        sync_all()
        start.record(stream)
        step_fn(args.steps)
        end.record(stream)
        torch.cuda.synchronize()
        sync_all()
    ms = start.elapsed_time(end)
    if dist is not None:
        red_dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([ms], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nf = torch.tensor([n_fn_rank], device=red_dev, dtype=torch.float64)
        dist.all_reduce(nf)
        n_fn_total = int(nf.item())
    else:
        n_fn_total = n_fn_rank
    # divergence / neighbour-timeout checks outside the timed region; the |u|
    # guard is a diagnostic: its trips are reported in the
    # line (the no-slip ring decelerates the u = 0.04 start, and the
    # pressure waves it launches overshoot 0.05 near the walls)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        runner.slab.solver.check()
    guard_trips = len(runner.slab.solver.guard_iterations)
    if runner.ipc is not None:
        runner.ipc.check()

    ms_step = ms / args.steps
    value = n_fn_total * args.steps / (ms / 1e3) / 1e6
    n_d = 8 if args.precision == "f64" else 4
    b_node = txmodel.b_node(19, n_d)
    alg_bytes = n_fn_rank * b_node
    achieved = alg_bytes / (ms_step / 1e3) / 1e9
    peak, peak_src = peaks()
    key = f"channel{args.edge}_{args.precision}_{args.table}"
    traffic = traffic_from_profiles(key)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"channel{args.edge}_periodic_{args.precision}"
                               + (f"_slab_x{world}" if world > 1 else ""),
                   "geometry": f"square channel d={args.edge} along z, BB ring, periodic z, "
                               f"{args.edge}x{args.edge}x{args.edge} per GPU"
                               + (f", global {args.edge}x{args.edge}x{args.edge * world}"
                                  if world > 1 else ""),
                   "model": "LBGK incompressible, tau=0.6", "layout_table": args.table,
                   "arithmetic": args.arith,
                   "n_fn_per_gpu": n_fn_rank, "t_n_per_gpu": n_fn_rank // 64,
                   "l2": "inputs larger than L2 (field %.2f GB per copy)"
                         % (n_fn_rank / 64 * 19 * 64 * n_d / 1e9),
                   "parallelism": f"slab{world}" if world > 1 else "single",
                   "u_guard_trips": guard_trips,
                   "halo": args.transport_used if world > 1 else None,
                   "shared_gpu_test_mode": bool(shared)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_node": b_node,
                     "metadata_bytes_per_launch": txmodel.metadata_bytes(n_fn_rank // 64),
                     "peak_source": peak_src, "frac_of_8TBs_spec": achieved / 8000.0},
        "clocks": clocks.report(),
        "gpu_launches": args.steps * runner.launches_per_step(),
    }
    if not args.no_e2e:
        if runner.ipc is not None:
            runner.ipc.close()
        del runner
        torch.cuda.empty_cache()
        line["e2e"] = e2e_run(args, torch, workloads.channel_z(args.edge, args.edge * world), world,
                              rank, dist)
    if rank == 0 and world == 1 and not args.no_sweep:
        line["porosity"] = porosity_block(args, torch)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_mlups(args.precision, args.edge, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

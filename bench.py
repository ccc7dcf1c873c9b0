"""Benchmark of the tiled D3Q19 LBGK step on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload auto|channel|dense_weak|vessel_strong]

Workloads (one "step" = one collide+propagate pass over every owned tile):
  channel        N = 1 default, BASELINE config 2: dense square channel
                 256^3, bounce-back ring, periodic along z, LBGK
                 incompressible, fp64, tau = 0.6, from a perturbed
                 equilibrium (u = 0.02 along z; paper_1611_02445_b200/
                 workloads.py).  The field (2 x 2.55 GB) is far larger than
                 L2 (126 MB), so no flush is needed.
  dense_weak     N > 1 default, BASELINE config 5 dense: weak scaling with a
                 1024 x 1024 x 128 z-slab per GPU of a 1024 x 1024 x 128N
                 channel periodic in z (N = 8: dense 1024^3, 40.8 GB of fp64
                 fields per GPU).  Boundary tile layers store their outgoing
                 z planes straight into the neighbours' ghost tiles over
                 NVLink peer memory, overlapped with the interior launch
                 (paper_1611_02445_b200/slabs.py).
  vessel_strong  BASELINE config 5 sparse: the 1024 x 1024 x 2048 vessel tree
                 (2048 x 1024^2 voxels, z longest so slab faces are 256 x 256
                 tiles), fixed total work over N GPUs (strong scaling).

Reported (one JSON line on rank 0):
  value      MLUPS over all ranks (non-solid node updates / s / 1e6), device
             time from CUDA events on the launching stream, max over ranks
  roofline   algorithmic bytes per launch = n_fn x 2 x 19 x 8 B (txmodel
             b_node) / average step time, vs MEASURED_PEAKS.json hbm_gbs;
             traffic = ncu dram bytes per launch from profiles/
             roofline_traffic.json, used only while its recorded hash of the
             kernel sources equals the current one (else null, "stale")
  e2e        the same metric through the public API from host data: geometry
             upload, device tiling, init, K steps each followed by an async
             D2H of the step's status word, final rho/u readout to the host
  porosity   "vs porosity" (rank 0, N = 1): BASELINE config 3 (256^3 sphere
             packs, d = 40, seed 1234, porosity 0.2 ... 1.0) in fp64 and fp32
             for the paper's block storage and the compact store, the
             storage="auto" pick, and config 4 (vessel tree 512x512x1024)
  scale_unit the per-GPU unit of the N > 1 default (dense 1024x1024x128) timed
             on one GPU, so E(N) can be read against the same work per GPU
  cpu_baseline  the C oracle (oracle/tlbm_oracle.c, OpenMP on all host cores)
             on the same 256^3 channel (rank 0, N = 1), plus the BASELINE.md
             plan number: the numpy oracle step on cavity 64^3 on 1 core
  --impl reference  times that same CPU oracle as the reference arm
"""

import argparse
import hashlib
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
WORKLOADS = ("auto", "channel", "dense_weak", "vessel_strong")
# sources that make up the step kernel (the ncu traffic figure is keyed to them)
KERNEL_SOURCES = ("Makefile", "paper_1611_02445_b200/csrc/common.cuh",
                  "paper_1611_02445_b200/csrc/d3q19.cuh",
                  "paper_1611_02445_b200/csrc/physics.cuh",
                  "paper_1611_02445_b200/csrc/step_impl.cuh",
                  "paper_1611_02445_b200/csrc/step_compact.cuh",
                  "paper_1611_02445_b200/csrc/mrt_pattern.cuh",
                  "paper_1611_02445_b200/csrc/step.cu",
                  "paper_1611_02445_b200/csrc/step_f64.cu",
                  "paper_1611_02445_b200/csrc/step_f32.cu")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--precision", default="f64", choices=["f64", "f32"])
    p.add_argument("--workload", default="auto", choices=WORKLOADS,
                   help="auto = channel at N = 1, dense_weak at N > 1")
    p.add_argument("--edge", type=int, default=256, help="channel edge in nodes")
    p.add_argument("--scale-edge", type=int, default=1024,
                   help="dense_weak cross-section edge in nodes")
    p.add_argument("--scale-length", type=int, default=128,
                   help="dense_weak z length per GPU in nodes")
    p.add_argument("--vessel-shape", default="1024,1024,2048")
    p.add_argument("--table", default="b200")
    p.add_argument("--arith", default="reference", choices=["reference", "fma"],
                   help="collision arithmetic: reference = bit-exact unfused order, "
                        "fma = fused multiply-adds (parity within tolerance)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-sweep", action="store_true",
                   help="skip the porosity block and the scale unit")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--transport", default="ipc", choices=["ipc", "nccl", "gloo"],
                   help="N>1 halo: ipc = fused peer stores from the step kernel (default), "
                        "nccl = pack + NCCL send/recv + unpack, gloo = host-staged (tests)")
    a = p.parse_args()
    if a.workload == "auto":
        a.workload = "channel" if a.gpus == 1 else "dense_weak"
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def kernel_source_hash():
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        with open(os.path.join(ROOT, rel), "rb") as fh:
            h.update(rel.encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def traffic_from_profiles(key):
    """(dram bytes per launch, note) from profiles/roofline_traffic.json when
    the entry was captured on the current kernel sources, else (None, why)."""
    path = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if not os.path.exists(path):
        return None, "no capture"
    e = json.load(open(path)).get(key)
    if not isinstance(e, dict):
        return None, f"no capture for {key}"
    cur = kernel_source_hash()
    if e.get("src_sha") != cur:
        return None, f"stale: captured on kernel sources {e.get('src_sha')}, now {cur}"
    return float(e["traffic"]), f"ncu --set full, {e.get('capture', '')}"


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


# ---------------------------------------------------------------- workloads
def vessel_shape(args):
    return tuple(int(v) for v in args.vessel_shape.split(","))


def workload(args, world, device=None):
    """(global geometry, config label, description, scaling, start velocity)."""
    from paper_1611_02445_b200 import workloads
    p = args.precision
    if args.workload == "channel":
        e = args.edge
        geo = workloads.channel_z(e, e * world)
        return (geo, f"channel{e}_periodic_{p}" + (f"_slab_x{world}" if world > 1 else ""),
                f"square channel d={e} along z, BB ring, periodic z, {e}x{e}x{e} per GPU"
                + (f", global {e}x{e}x{e * world}" if world > 1 else ""), "weak",
                (0.0, 0.0, 0.02))
    if args.workload == "dense_weak":
        e, ln = args.scale_edge, args.scale_length
        geo = workloads.channel_z(e, ln * world)
        return (geo, f"dense{e}x{e}x{ln}_per_gpu_weak_{p}",
                f"BASELINE config 5 dense: square channel d={e}, BB ring, periodic z, "
                f"{e}x{e}x{ln} per GPU, global {e}x{e}x{ln * world}", "weak", (0.0, 0.0, 0.02))
    shape = vessel_shape(args)
    geo = workloads.vessel_tree(shape, device=device)
    return (geo, f"vessel{'x'.join(map(str, shape))}_strong_{p}",
            f"BASELINE config 5 sparse: vessel tree {shape[0]}x{shape[1]}x{shape[2]} "
            f"(inlet z=0, outlet z={shape[2] - 1}), split over {world} GPU(s)", "strong",
            (0.0, 0.0, 0.01))


# ---------------------------------------------------------------- CPU oracle
def _oracle_channel(precision, edge, cores):
    from oracle import c_oracle, dense
    from paper_1611_02445_b200 import workloads
    dt = np.float64 if precision == "f64" else np.float32
    geo = workloads.channel_z(edge)
    f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.02))
    o = c_oracle.DenseOracle(geo.types, "incompressible", workloads.TAU, periodic=geo.periodic,
                             f0=f0, dtype=dt, nthreads=cores)
    return o, geo.nonsolid_count()


def cpu_oracle_mlups(precision, edge, seconds):
    """C oracle (OpenMP on all available host cores) on the full config-2
    channel edge^3, the same workload as the GPU headline: as many steps as
    fit in ``seconds`` (at least 3)."""
    cores = len(os.sched_getaffinity(0))
    o, n_fn = _oracle_channel(precision, edge, cores)
    o.run(1)                                     # warm-up (page faults, threads)
    steps, t0 = 0, time.perf_counter()
    while True:
        o.run(1)
        steps += 1
        el = time.perf_counter() - t0
        if (el >= seconds and steps >= 3) or steps >= 200:
            break
    return {"value": n_fn * steps / el / 1e6, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"C oracle (oracle/tlbm_oracle.c, OpenMP x{cores}) on the full channel "
                      f"{edge}^3 (periodic z), {precision}, {steps} steps in {el:.1f} s"}


def cpu_numpy_plan(steps=6):
    """BASELINE.md's CPU plan: the numpy step (oracle/dense.py: the
    reference's collide_lbgk / zou_he / reflect arithmetic composed per
    SURVEY Appendix A) on cavity 64^3, fp64, one core (numpy elementwise
    arithmetic is single-threaded)."""
    from oracle import dense
    from paper_1611_02445_b200 import workloads
    geo = workloads.cavity(64)
    f = dense.init_equilibrium(geo.shape, "incompressible", np.float64)
    kw = dict(inlet_velocity=geo.inlet_velocity, outlet_density=geo.outlet_density)
    f = dense.step(f, geo.types, "incompressible", workloads.TAU, **kw)      # warm-up
    t0 = time.perf_counter()
    for _ in range(steps):
        f = dense.step(f, geo.types, "incompressible", workloads.TAU, **kw)
    el = time.perf_counter() - t0
    n_fn = geo.nonsolid_count()
    return {"value": n_fn * steps / el / 1e6, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"numpy oracle step (oracle/dense.py) on cavity 64^3, f64, {steps} steps "
                      f"in {el:.1f} s (BASELINE.md CPU plan)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import c_oracle, dense
    from paper_1611_02445_b200 import workloads
    dt = np.float64 if args.precision == "f64" else np.float32
    cores = len(os.sched_getaffinity(0))
    if args.workload == "channel" and world == 1:
        o, n_fn = _oracle_channel(args.precision, args.edge, cores)
        label = f"channel{args.edge}_periodic_{args.precision}"
        sample = (f"the full channel {args.edge}^3 (periodic z) per step, the GPU arm's "
                  f"N = 1 workload")
    else:
        # bounded sample of a multi-GPU workload: a 16-layer z-slab of it
        # (per-node work is the same along z), periodic in z
        geo, label, _, _, _ = workload(args, world, device=None) \
            if args.workload != "vessel_strong" else (None, None, None, None, None)
        if geo is None:
            from paper_1611_02445_b200 import geometry
            shape = vessel_shape(args)
            full = geometry.generate_vessel_tree(shape)
            z0 = shape[2] // 2
            geo = geometry.Geometry(np.ascontiguousarray(full.types[:, :, z0:z0 + 16]),
                                    full.inlet_velocity, full.outlet_density)
            label = f"vessel{'x'.join(map(str, shape))}_strong_{args.precision}"
        else:
            geo = workloads.channel_z(geo.shape[0], 16)
        f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.02))
        o = c_oracle.DenseOracle(geo.types, "incompressible", workloads.TAU,
                                 geo.inlet_velocity, geo.outlet_density, periodic=geo.periodic,
                                 f0=f0, dtype=dt, nthreads=cores)
        n_fn = geo.nonsolid_count()
        sample = (f"a {geo.shape[0]}x{geo.shape[1]}x{geo.shape[2]} z-slab of the "
                  f"{args.workload} workload per step ({n_fn} non-solid nodes)")
    for _ in range(args.warmup):
        o.run(1)
    t_all = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        o.run(1)
        t_all.append(time.perf_counter() - t0)
    total = sum(t_all)
    value = n_fn * args.steps / total / 1e6
    sample = (f"C oracle port (oracle/tlbm_oracle.c, OpenMP x{cores}): {sample}, "
              f"{args.precision}; the reference has no step of its own (SURVEY 0.2)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "vessel_strong" else "weak",
            "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
            "config": {"workload": label, "sample_nodes": n_fn},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def e2e_run(args, torch, geo_host, world, rank, dist, u0):
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
    # the job's input -- the voxel tags -- in pinned host memory, like the
    # status and rho/u buffers (allocated outside the timed region)
    tags = torch.empty(geo_host.shape, dtype=torch.uint8, pin_memory=True)
    tags.numpy()[...] = geo_host.types
    geo_host = type(geo_host)(tags.numpy(), geo_host.inlet_velocity, geo_host.outlet_density,
                              periodic=geo_host.periodic)
    pinned = torch.empty(max(args.steps, args.warmup), dtype=torch.int32, pin_memory=True)
    rho = torch.empty((t_own, 64), dtype=dt, pin_memory=True)
    u = torch.empty((3, t_own, 64), dtype=dt, pin_memory=True)
    # one untimed pass of the whole e2e path with `warmup` steps first: a
    # serving process has its CUDA context, modules and caching-allocator
    # blocks already; the timed pass then measures the per-job work, not
    # first-use cudaMalloc of the field store
    _e2e_pass(args, torch, geo_host, world, rank, dist, cfg, pinned, rho, u, args.warmup, u0)
    el, t0, t1, t2, t3, n_fn, h2d, d2h = _e2e_pass(args, torch, geo_host, world, rank, dist, cfg,
                                                   pinned, rho, u, args.steps, u0)
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


def _e2e_pass(args, torch, geo_host, world, rank, dist, cfg, pinned, rho, u, steps, u0):
    from paper_1611_02445_b200 import slabs
    from paper_1611_02445_b200 import solver as sv
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run = slabs.DistributedSlabRunner(geo_host, world, rank, cfg,
                                      transport=getattr(args, "transport_used", args.transport),
                                      initial=(1.0, u0))
    s = run.slab.solver
    run.exchange_current()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for i in range(steps):
        run.step(1, check=False)
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


def _time_solver(torch, s, steps, warmup=3):
    s.step(warmup, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.step(steps, check=False)
    e1.record()
    torch.cuda.synchronize()
    s.check()
    return e0.elapsed_time(e1) / steps


def porosity_block(args, torch, steps=20,
                   porosities=(0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0)):
    """BASELINE configs 3 and 4: per geometry and precision, MLUPS and
    BU = MLUPS x B_node / peak for the paper's block storage ("blocks"), the
    compact store with the tile-parallel step ("compact") and with the
    node-parallel step ("nodes") -- CUDA events over `steps` launches after 3
    warm-up launches -- and the kernel storage="auto" picks (its number is
    that kernel's)."""
    from paper_1611_02445_b200 import workloads
    from paper_1611_02445_b200.solver import DeviceTiling, SimulationConfig, Solver
    from paper_1611_02445_b200.solver import resolve_auto_storage, use_nodes
    peak, _ = peaks()
    cases = [(f"{p:.1f}", workloads.sphere_pack(p, n=args.edge)) for p in porosities]
    cases.append(("vessel512x512x1024", workloads.vessel_tree((512, 512, 1024))))
    out = {"workload": f"sphere pack {args.edge}^3, d=40, seed 1234 (porosity 1.0: all-fluid "
                       "box) and vessel tree 512x512x1024 (seed 1234); LBGK incompressible",
           "kernels": {"blocks": "paper's 64-slot blocks, tile-parallel step",
                       "compact": "compact store, tile-parallel step",
                       "nodes": "compact store, node-parallel step"},
           "porosity": list(porosities), "eta_t": [], "vessel": {}}
    kernels = (("blocks", "blocks", "tile"), ("compact", "compact", "tile"),
               ("nodes", "compact", "nodes"))
    keys = [f"{m}_{k}" for k, _, _ in kernels for m in ("mlups", "bu")]
    for prec in ("f64", "f32"):
        out[prec] = {k: [] for k in keys + ["kernel_auto", "mlups_auto", "bu_auto"]}
    for name, geo in cases:
        tl = DeviceTiling(geo)
        ves = name.startswith("vessel")
        if ves:
            out["vessel"] = {"porosity": round(geo.porosity(), 4),
                             "eta_t": round(tl.n_fn / (64 * tl.t_n), 4), "t_n": tl.t_n}
        else:
            out["eta_t"].append(round(tl.n_fn / (64 * tl.t_n), 4))
        for prec in ("f64", "f32"):
            b_node = 2 * 19 * (8 if prec == "f64" else 4)
            rec = {}
            for kname, storage, trav in kernels:
                cfg = SimulationConfig(tau=workloads.TAU, precision=prec, u_max_guard=0.0,
                                       storage=storage)
                s = Solver(geo, cfg, tiling=tl, traversal=trav)
                ms = _time_solver(torch, s, steps)
                mlups = s.n_fn / (ms / 1e3) / 1e6
                rec[kname] = (round(mlups, 1), round(mlups * 1e6 * b_node / (peak * 1e9), 4))
                del s
                torch.cuda.empty_cache()
            acfg = resolve_auto_storage(SimulationConfig(precision=prec, storage="auto"),
                                        tl.n_fn, tl.t_n)
            auto = acfg.storage
            if auto == "compact":
                auto = "nodes" if use_nodes(acfg, tl.n_fn, tl.t_n, "auto") else "compact"
            d = out[prec] if not ves else out["vessel"].setdefault(prec, {})
            for kname, _, _ in kernels:
                for i, m in enumerate(("mlups", "bu")):
                    if ves:
                        d[f"{m}_{kname}"] = rec[kname][i]
                    else:
                        d[f"{m}_{kname}"].append(rec[kname][i])
            if ves:
                d.update(kernel_auto=auto, mlups_auto=rec[auto][0], bu_auto=rec[auto][1])
            else:
                d["kernel_auto"].append(auto)
                d["mlups_auto"].append(rec[auto][0])
                d["bu_auto"].append(rec[auto][1])
        del tl
        torch.cuda.empty_cache()
    return out


def scale_unit(args, torch, steps=20):
    """The per-GPU work of the N > 1 default (dense_weak) on one GPU, from
    the same perturbed start, so that the driver's E(N) compares like with
    like."""
    from paper_1611_02445_b200 import workloads
    e, ln = args.scale_edge, args.scale_length
    s = workloads.make_solver(workloads.channel_z(e, ln), args.precision,
                              u0=(0.0, 0.0, 0.02), table=args.table)
    ms = _time_solver(torch, s, steps)
    mlups = s.n_fn / (ms / 1e3) / 1e6
    peak, _ = peaks()
    b_node = 2 * 19 * (8 if args.precision == "f64" else 4)
    out = {"workload": f"dense{e}x{e}x{ln} (square channel, periodic z), one GPU",
           "n_fn": s.n_fn, "ms_per_step": ms, "mlups": mlups,
           "bu": mlups * 1e6 * b_node / (peak * 1e9),
           "field_gb": s.store.flat.numel() * s.store.flat.element_size() / 1e9}
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


def _gather(dist, torch, value, backend):
    """All ranks' float ``value`` as a list (rank order)."""
    if dist is None:
        return [value]
    dev = "cuda" if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(v.item()) for v in out]


def run_b200(args):
    import torch
    from paper_1611_02445_b200 import txmodel

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
    geo, label, desc, scaling, u0 = workload(args, world, device=local)
    transport = args.transport
    kw = dict(precision=args.precision, table=args.table, arithmetic=args.arith, u0=u0)
    try:
        runner = slabs.SlabWorkload(geo, world, rank, transport=transport, **kw)
    except RuntimeError as exc:
        if transport != "ipc":
            raise
        print(f"[bench] ipc halo unavailable ({exc}); falling back to nccl", file=sys.stderr)
        transport = "nccl" if backend == "nccl" else "gloo"
        runner = slabs.SlabWorkload(geo, world, rank, transport=transport, **kw)
    args.transport_used = transport
    n_fn_rank = runner.n_fn_owned
    t_own = runner.slab.own[1] - runner.slab.own[0]
    sync_all = runner.barrier

    for _ in range(args.warmup):
        runner.step(1, check=False)
    torch.cuda.synchronize()
    runner.check()
    sync_all()

    stream = torch.cuda.current_stream()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        sync_all()
        start.record(stream)
        runner.step(args.steps, check=False)
        end.record(stream)
        torch.cuda.synchronize()
        sync_all()
    ms = start.elapsed_time(end)
    # divergence / neighbour-timeout checks outside the timed region; the |u|
    # guard is a diagnostic: its trips are reported
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        runner.check()
    guard_trips = len(runner.slab.solver.guard_iterations)
    ms_all = _gather(dist, torch, ms, backend)
    nfn_all = _gather(dist, torch, n_fn_rank, backend)
    mem_all = _gather(dist, torch, torch.cuda.max_memory_allocated(local) / 1e9, backend)
    halo_all = _gather(dist, torch, runner.halo_bytes_per_step() if world > 1 else 0, backend)
    ms = max(ms_all)
    n_fn_total = int(sum(nfn_all))

    ms_step = ms / args.steps
    value = n_fn_total * args.steps / (ms / 1e3) / 1e6
    n_d = 8 if args.precision == "f64" else 4
    b_node = txmodel.b_node(19, n_d)
    alg_bytes = n_fn_rank * b_node
    achieved = alg_bytes / (ms_step / 1e3) / 1e9
    peak, peak_src = peaks()
    traffic, traffic_note = traffic_from_profiles(f"{label}_{args.table}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": label, "geometry": desc,
                   "model": "LBGK incompressible, tau=0.6", "layout_table": args.table,
                   "arithmetic": args.arith,
                   "n_fn_per_gpu": n_fn_rank, "t_n_per_gpu": t_own,
                   "n_fn_total": n_fn_total,
                   "l2": "inputs larger than L2 (field %.2f GB per copy per GPU)"
                         % (runner.slab.solver.t_n * 19 * 64 * n_d / 1e9),
                   "parallelism": f"slab{world}" if world > 1 else "single",
                   "u_guard_trips": guard_trips,
                   "halo": args.transport_used if world > 1 else None,
                   "halo_bytes_sent_per_step_per_rank": halo_all if world > 1 else None,
                   "memory_gb_per_rank": [round(v, 2) for v in mem_all],
                   "ms_per_step_per_rank": [v / args.steps for v in ms_all],
                   "shared_gpu_test_mode": bool(shared)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": traffic_note,
                     "kernel_src_sha": kernel_source_hash(),
                     "algorithmic_bytes_per_launch": alg_bytes,
                     "bytes_per_node": b_node,
                     "metadata_bytes_per_launch": txmodel.metadata_bytes(t_own),
                     "peak_source": peak_src, "frac_of_8TBs_spec": achieved / 8000.0},
        "clocks": clocks.report(),
        "gpu_launches": args.steps * runner.launches_per_step(),
    }
    if runner.ipc is not None:
        runner.ipc.close()
    del runner
    torch.cuda.empty_cache()
    if not args.no_e2e:
        line["e2e"] = e2e_run(args, torch, geo, world, rank, dist, u0)
    if rank == 0 and world == 1 and not args.no_sweep:
        line["porosity"] = porosity_block(args, torch)
        line["scale_unit"] = scale_unit(args, torch)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_mlups(args.precision, args.edge, args.cpu_seconds)
        line["cpu_baseline"]["plan_numpy_1core"] = cpu_numpy_plan()
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

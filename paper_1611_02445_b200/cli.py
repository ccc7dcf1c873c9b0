"""Command-line front end (the reference's pyproject entry
point ``tilelbm.cli:main`` has no module behind it).

    python -m paper_1611_02445_b200 run --geometry cavity:48 --iters 2000 --vtk out.vtk
    python -m paper_1611_02445_b200 bench --geometry cavity:100 --variant full --reps 100 \\
        --ref-bandwidth 6533.5
    python -m paper_1611_02445_b200 tile-stats --channel square:8
    python -m paper_1611_02445_b200 count-tx --precision f64 --layout optimized
    python -m paper_1611_02445_b200 info

Geometry mini-language: cavity:N, channel:square|circle:d:off1:off2:len[:ends],
spheres:n:diam:porosity:seed, box:n, vessel:nx:ny:nz, file:path (TLBM1).
Exit codes: 0 ok, 2 usage, 3 divergence, 4 I/O, 5 runtime (no CUDA device,
library error, invalid configuration).
"""

import argparse
import json
import sys

EXIT_OK, EXIT_USAGE, EXIT_DIVERGED, EXIT_IO, EXIT_RUNTIME = 0, 2, 3, 4, 5


class UsageError(ValueError):
    pass


def parse_geometry(spec):
    from . import geometry as g, workloads
    kind, _, rest = spec.partition(":")
    a = rest.split(":") if rest else []
    try:
        if kind == "cavity":
            return g.generate_cavity3d(int(a[0]))
        if kind == "channel":
            shape, d = a[0], int(a[1])
            off = (int(a[2]), int(a[3])) if len(a) > 3 else (0, 0)
            length = int(a[4]) if len(a) > 4 else 16
            ends = a[5] if len(a) > 5 else "wall"
            return g.generate_channel(shape, d, axis=0, offsets=off, length=length, ends=ends,
                                      inlet_velocity=(0.01, 0.0, 0.0))
        if kind == "spheres":
            return g.generate_sphere_pack(int(a[0]), float(a[1]), float(a[2]), int(a[3]),
                                          inlet_velocity=(0.0, 0.0, 0.01),
                                          device=workloads.generator_device())
        if kind == "box":
            return g.generate_box(int(a[0]), inlet_velocity=(0.0, 0.0, 0.01))
        if kind == "vessel":
            return g.generate_vessel_tree(tuple(int(v) for v in a[:3]),
                                          device=workloads.generator_device())
        if kind == "file":
            return g.load_voxels_path(rest)
    except (IndexError, ValueError) as exc:
        if isinstance(exc, OSError):
            raise
        raise UsageError(f"bad geometry spec {spec!r}: {exc}") from None
    raise UsageError(f"unknown geometry kind {kind!r}")


def _config(args):
    from .solver import SimulationConfig
    return SimulationConfig(collision=args.model, fluid=args.fluid, tau=args.tau,
                            precision=args.precision, table=args.layout,
                            arithmetic=args.arith, storage=args.storage)


def cmd_run(args):
    from . import solver
    geo = parse_geometry(args.geometry)
    outputs = {"vtk": args.vtk, "csv": args.csv, "checkpoint": args.checkpoint,
               "convergence_every": args.convergence_every, "tolerance": args.tolerance}
    _, diag = solver.run(_config(args), geo, args.iters, outputs=outputs,
                         resume_from=args.resume,
                         graph={"auto": "auto", "on": True, "off": False}[args.graph])
    print(json.dumps(diag))
    return EXIT_OK


def cmd_bench(args):
    """Per-launch timing with CUDA events (repeated launches)."""
    import torch

    from . import _native as nat
    from .solver import Solver
    geo = parse_geometry(args.geometry)
    s = Solver(geo, _config(args))
    variant = {"full": nat.FULL, "prop": nat.PROPAGATION_ONLY,
               "rw": nat.READ_WRITE_ONLY}[args.variant]
    s.step(args.warmup, variant=variant)
    times = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.step(1, variant=variant, check=False)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    s.check()
    mean = sum(times) / len(times)
    b_node = 304 if args.precision == "f64" else 152
    mflups = s.n_fn / mean / 1e6
    row = {"geometry": args.geometry, "variant": args.variant, "model": args.model,
           "precision": args.precision, "reps": args.reps, "mean_s": mean, "min_s": min(times),
           "max_s": max(times), "mflups": mflups, "n_fn": s.n_fn, "t_n": s.t_n}
    if args.ref_bandwidth:
        row["bandwidth_utilization"] = mflups * 1e6 * b_node / (args.ref_bandwidth * 1e9)
    print(",".join(row))
    print(",".join(str(v) for v in row.values()))
    return EXIT_OK


def cmd_tile_stats(args):
    from . import tiling
    if args.channel:
        shape, d = args.channel.split(":")
        rows, mean = tiling.channel_tiling_sweep(shape, int(d))
        print("off1,off2,eta_t")
        for (o1, o2), eta in rows:
            print(f"{o1},{o2},{float(eta)}")
        print(f"mean,,{float(mean)}")
        return EXIT_OK
    geo = parse_geometry(args.geometry)
    grid = tiling.build_tiling(geo)
    st = tiling.tile_utilization(grid, geo)
    print("t_n,n_fn,eta_t,n_tfn,n_tsn,eta_f,eta_e")
    print(f"{st.t_n},{st.n_fn},{st.eta_t},{st.n_tfn},{st.n_tsn},{st.eta_f},{st.eta_e}")
    return EXIT_OK


def cmd_plan(args):
    """Size an N-GPU slab run on the host (no GPU needed)."""
    from . import slabs
    geo = parse_geometry(args.geometry)
    print(json.dumps(slabs.plan_run(geo, args.gpus, args.precision, args.storage,
                                    args.budget_gb)))
    return EXIT_OK


def cmd_count_tx(args):
    from . import layout, txmodel
    table = layout.LayoutTable(args.layout)
    rep = txmodel.count_tile_overheads(table, args.precision)
    print("direction,segments")
    for k, v in rep.per_direction_reads.items():
        print(f"{k},{v}")
    print(f"total,{rep.tile_read_total}")
    print(f"minimum,{rep.tile_read_min}")
    print(f"whole_tile_unit,{txmodel.count_tile_reads_whole_tile(table, args.precision)}")
    return EXIT_OK


def cmd_info(args):
    import torch

    from . import _native as nat
    lib = nat.load()
    info = {"abi": lib.tlbm_abi_version(), "library": nat.LIB_PATH,
            "cuda_available": torch.cuda.is_available()}
    if torch.cuda.is_available():
        p = torch.cuda.get_device_properties(0)
        info.update(device=p.name, sms=p.multi_processor_count,
                    memory_gb=p.total_memory / 1e9, cc=f"{p.major}.{p.minor}")
    print(json.dumps(info))
    return EXIT_OK


def build_parser():
    p = argparse.ArgumentParser(prog="paper_1611_02445_b200")
    sub = p.add_subparsers(dest="cmd", required=True)

    def sim_args(sp):
        sp.add_argument("--geometry", default="cavity:48")
        sp.add_argument("--model", default="lbgk", choices=["lbgk", "mrt"])
        sp.add_argument("--fluid", default="incompressible",
                        choices=["incompressible", "quasi-compressible"])
        sp.add_argument("--tau", type=float, default=0.6)
        sp.add_argument("--precision", default="f64", choices=["f64", "f32"])
        sp.add_argument("--layout", default=None, choices=["b200", "optimized", "xyz"],
                        help="default: b200 (blocks storage), xyz (compact)")
        sp.add_argument("--arith", default="reference", choices=["reference", "fma"])
        sp.add_argument("--storage", default="blocks", choices=["blocks", "compact", "auto"])

    r = sub.add_parser("run")
    sim_args(r)
    r.add_argument("--iters", type=int, default=1000)
    r.add_argument("--vtk")
    r.add_argument("--csv")
    r.add_argument("--convergence-every", type=int, default=0)
    r.add_argument("--tolerance", type=float)
    r.add_argument("--checkpoint", help="save the final state here (.npz)")
    r.add_argument("--resume", help="start from this checkpoint (same geometry)")
    r.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                   help="replay CUDA graphs of 64 steps (auto: small domains)")
    b = sub.add_parser("bench")
    sim_args(b)
    b.add_argument("--variant", default="full", choices=["full", "prop", "rw"])
    b.add_argument("--reps", type=int, default=100)
    b.add_argument("--warmup", type=int, default=3)
    b.add_argument("--ref-bandwidth", type=float, help="GB/s for bandwidth utilization")
    t = sub.add_parser("tile-stats")
    t.add_argument("--geometry", default="cavity:48")
    t.add_argument("--channel", help="square:d or circle:d -- the 16-offset sweep")
    c = sub.add_parser("count-tx")
    c.add_argument("--precision", default="f64", choices=["f64", "f32"])
    c.add_argument("--layout", default="optimized", choices=["b200", "optimized", "xyz"])
    pl = sub.add_parser("plan", help="per-rank tiles, memory and halo bytes of an N-GPU run")
    pl.add_argument("--geometry", default="cavity:48")
    pl.add_argument("--gpus", type=int, default=1)
    pl.add_argument("--precision", default="f64", choices=["f64", "f32"])
    pl.add_argument("--storage", default="blocks", choices=["blocks", "compact", "auto"])
    pl.add_argument("--budget-gb", type=float, default=179.0)
    sub.add_parser("info")
    return p


COMMANDS = {"run": cmd_run, "bench": cmd_bench, "tile-stats": cmd_tile_stats,
            "count-tx": cmd_count_tx, "plan": cmd_plan, "info": cmd_info}


def main(argv=None):
    from .collision import DivergenceError
    try:
        args = build_parser().parse_args(argv)
    except SystemExit as exc:
        return EXIT_USAGE if exc.code else EXIT_OK
    try:
        return COMMANDS[args.cmd](args)
    except UsageError as exc:
        print(f"usage error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except DivergenceError as exc:
        print(f"diverged at iteration {exc.iteration}: {exc}", file=sys.stderr)
        return EXIT_DIVERGED
    except OSError as exc:
        print(f"I/O error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (RuntimeError, ValueError) as exc:   # no CUDA device, library errors, bad config
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())

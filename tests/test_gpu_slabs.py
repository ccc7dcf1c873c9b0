"""GPU: the z-slab decomposition with device halo pack/unpack (virtual ranks
on one GPU) is bit-identical to the single-domain step."""

import numpy as np
import pytest
import torch

from oracle import dense
from paper_1611_02445_b200 import geometry, slabs, solver

pytestmark = pytest.mark.gpu
TILE = slabs.TILE


def _f0(geo, dt, seed=3):
    rng = np.random.default_rng(seed)
    f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.02))
    return f0 * (1 + rng.uniform(-1e-3, 1e-3, f0.shape)).astype(dt)


def _local_f(f0, r, nz):
    idx = []
    if r.lower >= 0:
        idx += [z % nz for z in range(r.z0 - TILE, r.z0)]
    idx += list(range(r.z0, r.z1))
    if r.upper >= 0:
        # a partial top layer (nz % 4 != 0) is a partial ghost; the wrap to
        # z = 0 happens only across a periodic seam (r.z1 == nz)
        hi = min(r.z1 + TILE, nz) if r.z1 < nz else r.z1 + TILE
        idx += [z % nz for z in range(r.z1, hi)]
    return np.ascontiguousarray(f0[..., idx])


CASES = {
    "pack_io": lambda: geometry.generate_sphere_pack(32, 8, 0.6, seed=9,
                                                     inlet_velocity=(0, 0, 0.02)),
    "chan_periodic": lambda: geometry.generate_channel("circle", 18, axis=2, offsets=(1, 2),
                                                       length=40, ends="periodic"),
    "cavity": lambda: geometry.generate_cavity3d(30),
}


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("world", [2, 3, 5, 8])   # cavity 30 at 8: partial last layer
@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_virtual_slabs_bit_identical(name, world, dt, fused):
    geo = CASES[name]()
    prec = "f64" if dt == np.float64 else "f32"
    cfg = solver.SimulationConfig(precision=prec, u_max_guard=0.0)
    f0 = _f0(geo, dt)
    ref = solver.Solver(geo, cfg)
    ref.set_fields_canonical(dense.to_canonical(f0, ref.tile_grid.non_empty, np.zeros(19)))
    steps = 12
    ref.step(steps)
    want = ref.to_dense(ref.fields_canonical(device=True))

    vs = slabs.VirtualSlabs(geo, world, cfg, fused=fused)
    nz = geo.shape[2]
    for sl in vs.slabs:
        s = sl.solver
        fl = _local_f(f0, sl.range, nz)
        s.set_fields_canonical(dense.to_canonical(fl, s.tile_grid.non_empty, np.zeros(19)))
    vs.step(steps)
    got = torch.zeros_like(want)
    for sl in vs.slabs:
        s = sl.solver
        d = s.to_dense(s.fields_canonical(device=True))
        lo = TILE if sl.range.lower >= 0 else 0
        got[..., sl.range.z0:sl.range.z1] = d[..., lo:lo + sl.range.z1 - sl.range.z0]
    mask = torch.from_numpy(geo.types != 0).cuda()
    assert torch.equal(got[:, mask], want[:, mask])
    assert sum(sl.n_fn_owned for sl in vs.slabs) == ref.n_fn


def test_initial_exchange_fills_ghosts():
    geo = CASES["chan_periodic"]()
    cfg = solver.SimulationConfig(u_max_guard=0.0)
    vs = slabs.VirtualSlabs(geo, 3, cfg)
    for r, sl in enumerate(vs.slabs):
        sl.solver.init_equilibrium(1.0 + 0.01 * r, (0.0, 0.0, 0.01))
    vs.exchange_current()
    # every ghost plane now holds the neighbour's owned values
    for sl in vs.slabs:
        s = sl.solver
        d = s.to_dense(s.fields_canonical(device=True))
        lower = vs.slabs[sl.range.lower].solver
        dl = lower.to_dense(lower.fields_canonical(device=True))
        # T direction (5) at ghost plane z=3 equals lower's top owned plane
        top_owned = TILE + (vs.slabs[sl.range.lower].range.z1
                            - vs.slabs[sl.range.lower].range.z0) - 1
        ns = torch.from_numpy(geo.types[:, :, 0] != 0).cuda()
        assert torch.equal(d[5, :, :, TILE - 1][ns], dl[5, :, :, top_owned][ns])


def test_slab_channel_single_rank_runs():
    run = slabs.SlabChannel(32, 1, 0)
    run.step(5)
    s = run.slab.solver
    s.check()
    assert run.n_fn_owned == 32 ** 3 and s.iteration == 5


COLLISIONS = {"lbgk": {}, "mrt": {"collision": "mrt"},
              "mrt_fma": {"collision": "mrt", "arithmetic": "fma"},
              "lbgk_fma_quasi": {"arithmetic": "fma", "fluid": "quasi-compressible"},
              "compact": {"storage": "compact"},
              "compact_f32_mrt": {"storage": "compact", "precision": "f32", "collision": "mrt"},
              "compact_nodes": {"storage": "compact", "traversal": "nodes"},
              "compact_nodes_f32_mrt": {"storage": "compact", "precision": "f32",
                                        "collision": "mrt", "traversal": "nodes"},
              "auto": {"storage": "auto"}}


def _split(coll):
    """SimulationConfig kwargs and the slab traversal of a COLLISIONS entry."""
    kw = dict(COLLISIONS[coll])
    return kw, kw.pop("traversal", "auto")


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("coll", [c for c in COLLISIONS if c != "lbgk"])
@pytest.mark.parametrize("name", ["pack_io", "chan_periodic"])
def test_virtual_slabs_collision_modes(name, coll, fused):
    """MRT, FMA arithmetic and compact storage through the slab
    decomposition (halo pack/unpack, or the fused peer stores): bit-identical
    to the single-domain step with the same configuration."""
    geo = CASES[name]()
    kw, trav = _split(coll)
    cfg = solver.SimulationConfig(u_max_guard=0.0, **kw)
    if cfg.storage == "auto":
        cfg = slabs.resolve_auto_storage_global(cfg, geo)
    f0 = _f0(geo, cfg.dtype)
    ref = solver.Solver(geo, cfg)
    ref.set_fields_canonical(dense.to_canonical(f0, ref.tile_grid.non_empty, np.zeros(19)))
    ref.step(8)
    want = ref.to_dense(ref.fields_canonical(device=True))
    vs = slabs.VirtualSlabs(geo, 3, cfg, fused=fused, traversal=trav)
    if trav == "nodes":
        assert all(sl.solver.nodes is not None for sl in vs.slabs)
    for sl in vs.slabs:
        s = sl.solver
        fl = _local_f(f0, sl.range, geo.shape[2])
        s.set_fields_canonical(dense.to_canonical(fl, s.tile_grid.non_empty, np.zeros(19)))
    vs.step(8)
    got = torch.zeros_like(want)
    for sl in vs.slabs:
        d = sl.solver.to_dense(sl.solver.fields_canonical(device=True))
        lo = TILE if sl.range.lower >= 0 else 0
        got[..., sl.range.z0:sl.range.z1] = d[..., lo:lo + sl.range.z1 - sl.range.z0]
    mask = torch.from_numpy(geo.types != 0).cuda()
    assert torch.equal(got[:, mask], want[:, mask])


def _mp_worker(rank, world, port, steps, out, transport="gloo", coll="lbgk"):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    geo = CASES["pack_io"]()
    kw, trav = _split(coll)
    cfg = solver.SimulationConfig(u_max_guard=0.0, **kw)
    run = slabs.DistributedSlabRunner(geo, world, rank, cfg, transport=transport,
                                      traversal=trav)
    s = run.slab.solver
    f0 = _f0(geo, np.float64)
    fl = _local_f(f0, run.slab.range, geo.shape[2])
    s.set_fields_canonical(dense.to_canonical(fl, s.tile_grid.non_empty, np.zeros(19)))
    if run.ipc is not None:
        run.exchange_current()
    run.step(steps)
    if run.ipc is not None:
        run.ipc.check()
    d = s.to_dense(s.fields_canonical(device=True))
    lo = TILE if run.slab.range.lower >= 0 else 0
    r = run.slab.range
    out[rank] = (r.z0, r.z1, d[..., lo:lo + r.z1 - r.z0].cpu().numpy())
    if run.ipc is not None:
        run.ipc.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("transport,coll", [("gloo", "lbgk"), ("ipc", "lbgk"), ("ipc", "mrt"),
                                            ("ipc", "mrt_fma"), ("ipc", "compact"),
                                            ("gloo", "compact"), ("ipc", "compact_nodes")])
@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_runner_on_one_gpu(world, transport, coll):
    """DistributedSlabRunner in `world` processes sharing cuda:0 == the
    single-domain step.  transport "gloo": halo staged through host memory;
    "ipc": the fused peer-store halo over CUDA IPC mappings with the
    stream-ordered step counters (the multi-GPU product path, here with all
    peers on one device)."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    steps = 10
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, steps, out, transport, coll))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    geo = CASES["pack_io"]()
    cfg = solver.SimulationConfig(u_max_guard=0.0, **_split(coll)[0])
    ref = solver.Solver(geo, cfg)
    ref.set_fields_canonical(dense.to_canonical(_f0(geo, np.float64), ref.tile_grid.non_empty,
                                                np.zeros(19)))
    ref.step(steps)
    want = ref.to_dense(ref.fields_canonical(device=True)).cpu().numpy()
    got = np.zeros_like(want)
    for rank in range(world):
        z0, z1, d = out[rank]
        got[..., z0:z1] = d
    mask = geo.types != 0
    assert np.array_equal(got[:, mask], want[:, mask])

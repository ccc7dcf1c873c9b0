"""CPU (gloo, world_size 2 and 3) check of the multi-GPU slab decomposition
logic: SlabPlan's cuts, ghost layers, neighbour ranks, periodic wrap and the
fixed send/recv post order of NcclHalo, driving the dense C oracle per rank.
The owned fields after N steps must equal the single-domain oracle bit for
bit.  (The device halo pack/unpack kernels are checked against the same
single-domain result on the GPU by tests/test_gpu_slabs.py.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1611_02445_b200 import geometry
from paper_1611_02445_b200.slabs import TILE, SlabPlan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _geometries():
    pack = geometry.generate_sphere_pack(16, 5, 0.7, seed=4, inlet_velocity=(0, 0, 0.02))
    chan = geometry.generate_channel("square", 10, axis=2, length=24, ends="periodic")
    # nz % 4 != 0 and one rank per tile layer: the last rank owns a partial
    # layer of 2 nodes, which is the upper ghost of the rank below
    cav = geometry.generate_cavity3d(10)
    return {"pack": pack, "chan": chan, "cav": cav}


def _initial(geo, dt=np.float64):
    from oracle import dense
    rng = np.random.default_rng(7)
    f0 = dense.init_equilibrium(geo.shape, "incompressible", dt, 1.0, (0.0, 0.0, 0.02))
    return f0 * (1 + rng.uniform(-1e-3, 1e-3, f0.shape))


def _worker(rank, world, port, name, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import c_oracle
    geo = _geometries()[name]
    plan = SlabPlan(geo, world)
    r = plan.ranges[rank]
    lgeo = plan.local_geometry(geo, rank)
    f0 = _initial(geo)
    # local dense field: the same slicing as the tags
    nz = geo.shape[2]
    idx = []
    if r.lower >= 0:
        idx += [(z % nz) for z in range(r.z0 - TILE, r.z0)]
    idx += list(range(r.z0, r.z1))
    n_hi = 0
    if r.upper >= 0:
        n_hi = min(TILE, nz - r.z1) if r.z1 < nz else TILE
        idx += [(z % nz) for z in range(r.z1, r.z1 + n_hi)]
    assert lgeo.shape[2] == len(idx)
    assert np.array_equal(lgeo.types, geo.types[:, :, idx])
    f = np.ascontiguousarray(f0[:, :, :, idx])
    lo = TILE if r.lower >= 0 else 0
    hi = f.shape[3] - n_hi
    n_own_lo = min(TILE, r.z1 - r.z0)             # what the lower rank's upper ghost holds
    for _ in range(steps):
        o = c_oracle.DenseOracle(lgeo.types, "incompressible", 0.6, geo.inlet_velocity,
                                 geo.outlet_density, periodic=lgeo.periodic, f0=f, nthreads=1)
        o.run(1)
        f = o.f.copy()
        # exchange whole boundary tile layers (dense analogue of the plane halo),
        # same post order as NcclHalo: sends [up, down], recvs [below, above]
        ops, recv_lo, recv_hi = [], None, None
        if r.upper >= 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(f[..., hi - TILE:hi].copy()),
                                  r.upper))
        if r.lower >= 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(f[..., lo:lo + n_own_lo].copy()),
                                  r.lower))
        if r.lower >= 0:
            recv_lo = torch.empty(f[..., :TILE].shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, recv_lo, r.lower))
        if r.upper >= 0:
            recv_hi = torch.empty(f[..., :n_hi].shape, dtype=torch.float64)
            ops.append(dist.P2POp(dist.irecv, recv_hi, r.upper))
        for q in dist.batch_isend_irecv(ops):
            q.wait()
        if recv_lo is not None:
            f[..., :TILE] = recv_lo.numpy()
        if recv_hi is not None:
            f[..., hi:] = recv_hi.numpy()
    out[rank] = (r.z0, r.z1, f[..., lo:hi].copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,world", [("pack", 2), ("chan", 2), ("chan", 3), ("pack", 3),
                                        ("cav", 3)])
def test_gloo_slab_decomposition_matches_single_domain(name, world):
    from oracle import c_oracle
    c_oracle.build()
    steps = 4
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, steps, out))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    geo = _geometries()[name]
    o = c_oracle.DenseOracle(geo.types, "incompressible", 0.6, geo.inlet_velocity,
                             geo.outlet_density, periodic=geo.periodic, f0=_initial(geo))
    o.run(steps)
    ns = geo.types != 0
    got = np.zeros_like(o.f)
    covered = np.zeros(geo.shape[2], dtype=int)
    for rank in range(world):
        z0, z1, f = out[rank]
        got[..., z0:z1] = f
        covered[z0:z1] += 1
    assert np.all(covered == 1)
    assert np.array_equal(got[:, ns], o.f[:, ns])


def test_plan_balances_fluid_nodes():
    g = geometry.generate_sphere_pack(64, 16, 0.5, seed=1)
    for world in (2, 4, 8):
        plan = SlabPlan(g, world)
        w = [plan.layer_weight[r.z0 // TILE:-(-r.z1 // TILE)].sum() for r in plan.ranges]
        assert plan.ranges[0].z0 == 0 and plan.ranges[-1].z1 == 64
        assert all(a.z1 == b.z0 for a, b in zip(plan.ranges, plan.ranges[1:]))
        assert max(w) - min(w) <= 2 * plan.layer_weight.max()
        assert plan.ranges[0].lower == -1 and plan.ranges[-1].upper == -1
    per = geometry.generate_channel("square", 8, axis=2, length=32, ends="periodic")
    plan = SlabPlan(per, 4)
    assert plan.ranges[0].lower == 3 and plan.ranges[3].upper == 0
    assert plan.local_types(per.types, 0).shape[2] == 8 + 2 * TILE


def test_plan_partial_last_layer_ghost():
    """nz % 4 != 0 with the last rank owning only the partial top layer: the
    rank below gets z = z1..nz-1 as its upper ghost, never the wrapped z = 0
    wall (slabs.py local_types)."""
    for n, world in ((10, 3), (30, 8)):
        g = geometry.generate_cavity3d(n)
        plan = SlabPlan(g, world)
        assert plan.ranges[-1].z1 == n and not plan.periodic_z
        for rk, r in enumerate(plan.ranges):
            lt = plan.local_types(g.types, rk)
            lo = r.z0 - TILE if r.lower >= 0 else r.z0
            hi = min(r.z1 + TILE, n) if r.upper >= 0 else r.z1
            assert np.array_equal(lt, g.types[:, :, lo:hi])


def test_plan_run_matches_decomposition():
    """slabs.plan_run (host-only sizing) agrees with the slab plan and the
    tile counts of the geometry."""
    import numpy as np
    from paper_1611_02445_b200 import geometry, slabs
    geo = geometry.generate_channel("square", 12, axis=2, length=40, ends="periodic")
    one = slabs.plan_run(geo, 1)
    t = geo.types != 0
    assert one["ranks"][0]["nonsolid_nodes"] == int(t.sum())
    assert one["ranks"][0]["tiles"] == 3 * 3 * 10 and one["fits"]      # 12 x 12 -> 3 x 3 tiles
    four = slabs.plan_run(geo, 4, precision="f32", storage="compact")
    owned = sum(r["z"][1] - r["z"][0] for r in four["ranks"])
    assert owned == 40 and four["storage"] == "compact"
    # periodic z: every rank has two ghost layers and two boundary layers
    assert all(r["tiles"] == 9 * ((r["z"][1] - r["z"][0]) // 4 + 2) for r in four["ranks"])
    assert all(r["halo_bytes_sent_received_per_step"] == 2 * 80 * 4 * 18 for r in four["ranks"])
    assert four["ranks"][0]["field_gb"] == round(2 * 19 * 4 * four["ranks"][0]["nonsolid_nodes"] / 1e9, 3)

"""BASELINE.json configurations as concrete synthetic inputs.

Seeds are fixed; tau = 0.6; LBGK incompressible unless noted.

cavity(64)          config 1: lid-driven cavity, lid u = (0.05, 0, 0)
channel(256)        config 2: square channel d = 256 along x, bounce-back
                    ring on the y/z faces, periodic in x (extension); started
                    from equilibrium(rho, u) with u = (0.04, 0, 0) and a seeded
                    +/-1e-3 perturbation of rho and u so the flow evolves
sphere_pack(p)      config 3: generate_sphere_pack(256, 40, p, seed=1234,
                    flow_axis=2, inlet u = (0, 0, 0.01)); p = 1.0 -> all-fluid
                    box with the same face typing
vessel_tree()       config 4: seeded bifurcating tube tree 512x512x1024
"""

import torch

from . import geometry
from .solver import SimulationConfig, Solver

TAU = 0.6


def cavity(b=64):
    return geometry.generate_cavity3d(b)


def channel(n=256, length=None):
    return geometry.generate_channel("square", n, axis=0, length=n if length is None else length,
                                     ends="periodic")


def channel_z(n=256, length=None):
    """The config-2 channel with its axis along z (the slab axis): n x n
    cross-section, periodic in z, ``length`` nodes long (default n)."""
    return geometry.generate_channel("square", n, axis=2, length=n if length is None else length,
                                     ends="periodic")


def generator_device(device="auto"):
    """The device the geometry generators run on: "auto" = cuda:0 when a GPU
    is present (bit-identical voxels either way), None = the host."""
    if device == "auto":
        return 0 if torch.cuda.is_available() else None
    return device


def sphere_pack(porosity, n=256, diameter=40, seed=1234, device="auto"):
    if porosity >= 1.0:
        return geometry.generate_box(n, flow_axis=2, inlet_velocity=(0.0, 0.0, 0.01))
    return geometry.generate_sphere_pack(n, diameter, porosity, seed, flow_axis=2,
                                         inlet_velocity=(0.0, 0.0, 0.01), outlet_density=1.0,
                                         device=generator_device(device))


def vessel_tree(shape=(512, 512, 1024), seed=1234, device="auto"):
    return geometry.generate_vessel_tree(shape, seed=seed, device=generator_device(device))


def perturbed_fields(t_n, dtype, device, u0=(0.04, 0.0, 0.0), amp=1e-3, seed=1234):
    """(rho, u) canonical fields: rho = 1 + e, u = u0 + e, e ~ U(-amp, amp)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    rho = 1.0 + amp * (2 * torch.rand((t_n, 64), generator=g, device=device, dtype=dtype) - 1)
    u = amp * (2 * torch.rand((3, t_n, 64), generator=g, device=device, dtype=dtype) - 1)
    for a in range(3):
        u[a] += u0[a]
    return rho, u


def make_solver(geo, precision="f64", fluid="incompressible", table=None, perturb=True,
                device=None, u0=(0.04, 0.0, 0.0), index64=False, arithmetic="reference",
                storage="blocks", traversal="auto"):
    cfg = SimulationConfig(fluid=fluid, tau=TAU, precision=precision, table=table,
                           arithmetic=arithmetic, storage=storage)
    s = Solver(geo, cfg, device=device, index64=index64, traversal=traversal)
    if perturb:
        rho, u = perturbed_fields(s.t_n, s.store.tdtype, s.device, u0)
        s.init_from_macroscopic(rho, u)
    return s

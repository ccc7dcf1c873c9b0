"""Wall reflection and Zou-He face closures (reference boundaries.py).

Boundary contract (boundaries.py:1-28), implemented inside the fused step:
missing pulls at any non-solid node take the node's own opposite population
(halfway bounce-back); BB_WALL nodes additionally reflect instead of
colliding; inlet/outlet nodes get the Zou-He closure of their unique domain
face and then collide.

The closure index sets (``FaceClosure``) are host metadata identical to the
reference's; the arithmetic of ``zou_he_velocity`` / ``zou_he_pressure`` runs
in libtlbm (csrc/physics.cuh) in the reference's order.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as nat
from .collision import FluidModel, _to_device, fluid_code
from .geometry import NodeType
from .lattice import E_VECTORS, OPPOSITE, Q


@dataclass
class FaceClosure:
    axis: int
    inward_sign: int
    unknown_axis: int
    unknown_axis_opp: int
    diagonals: tuple
    k0: tuple
    km: tuple
    tangential: dict

    @property
    def face_id(self):
        """Library face code 2*axis + (0 low | 1 high)."""
        return 2 * self.axis + (0 if self.inward_sign > 0 else 1)


def face_closure(axis, inward_sign):
    """Index sets of one axis-aligned face (boundaries.py:53-85)."""
    axis, inward_sign = int(axis), int(inward_sign)
    normal = np.zeros(3, dtype=np.int64)
    normal[axis] = inward_sign
    cn = E_VECTORS @ normal
    k0 = tuple(int(q) for q in np.flatnonzero(cn == 0))
    km = tuple(int(q) for q in np.flatnonzero(cn == -1))
    axis_dir, diagonals = None, []
    for q in np.flatnonzero(cn == 1):
        q = int(q)
        side = [a for a in range(3) if a != axis and E_VECTORS[q, a]]
        if side:
            diagonals.append((q, int(OPPOSITE[q]), side[0], int(E_VECTORS[q, side[0]])))
        else:
            axis_dir = q
    tangential = {tau: (tuple(q for q in k0 if E_VECTORS[q, tau] == 1),
                        tuple(q for q in k0 if E_VECTORS[q, tau] == -1))
                  for tau in range(3) if tau != axis}
    return FaceClosure(axis, inward_sign, axis_dir, int(OPPOSITE[axis_dir]),
                       tuple(diagonals), k0, km, tangential)


FACE_CLOSURES = {(a, s): face_closure(a, s) for a in range(3) for s in (1, -1)}


def classify_boundary_faces(geometry):
    """{(axis, inward_sign): (inlet_ids, outlet_ids)} with flat C-order node
    ids; rejects inlet/outlet nodes not on exactly one face
    (boundaries.py:95-129).  Periodic axes (extension) have no faces."""
    dev = nat.require_cuda()
    t = torch.from_numpy(geometry.types).to(dev)
    dims = torch.tensor(t.shape, device=dev)
    io = (t == NodeType.VELOCITY_INLET) | (t == NodeType.PRESSURE_OUTLET)
    ids = torch.nonzero(io.view(-1)).view(-1)
    if ids.numel() == 0:
        return {}
    coords = torch.stack(torch.unravel_index(ids, tuple(t.shape)), dim=1)
    per = torch.tensor(geometry.periodic, device=dev)
    on_low = (coords == 0) & ~per
    on_high = (coords == dims - 1) & ~per
    count = on_low.sum(1) + on_high.sum(1)
    bad = count != 1
    if bool(bad.any()):
        x, y, z = (int(v) for v in coords[int(torch.nonzero(bad)[0, 0])])
        raise ValueError(f"inlet/outlet node ({x}, {y}, {z}) does not lie on exactly one "
                         "axis-aligned domain face")
    flat = t.view(-1)
    out = {}
    for axis in range(3):
        for sign, mask in ((1, on_low[:, axis]), (-1, on_high[:, axis])):
            sel = ids[mask]
            if sel.numel() == 0:
                continue
            tags = flat[sel]
            out[(axis, sign)] = (sel[tags == NodeType.VELOCITY_INLET].cpu().numpy(),
                                 sel[tags == NodeType.PRESSURE_OUTLET].cpu().numpy())
    return out


def _zou_he(g, closure, kind, u, rho0, model):
    gt, as_np = _to_device(g)
    if gt.dim() != 2 or gt.shape[0] != Q:
        raise ValueError("expected gathered populations of shape (19, m)")
    m = int(gt.shape[1])
    ret = torch.empty(m, dtype=gt.dtype, device=gt.device)
    ux, uy, uz = (float(c) for c in u)
    nat.call("tlbm_zou_he", nat.ptr(gt), nat.code_of(gt.dtype), fluid_code(model),
             closure.face_id, kind, m, ux, uy, uz, float(rho0), nat.ptr(ret),
             nat.stream_ptr(gt.device))
    if as_np:
        g[...] = gt.cpu().numpy()      # in place, like the reference
        return ret.cpu().numpy()
    if gt.data_ptr() != g.data_ptr():
        g.copy_(gt)
    return ret


def zou_he_velocity(g, closure, u, model=FluidModel.INCOMPRESSIBLE):
    """Velocity inlet, in place on g (19, m); returns the implied density
    (boundaries.py:139-157)."""
    return _zou_he(g, closure, 0, u, 1.0, model)


def zou_he_pressure(g, closure, rho0, model=FluidModel.INCOMPRESSIBLE):
    """Pressure outlet, in place on g (19, m); returns the normal momentum
    (boundaries.py:160-176)."""
    return _zou_he(g, closure, 1, (0.0, 0.0, 0.0), rho0, model)

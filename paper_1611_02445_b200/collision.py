"""Node physics API on the GPU: moments, equilibrium, LBGK collision.

Same names, shapes and dtype behaviour as ``tilelbm.collision``
(collision.py:28-130, 250-252); the arithmetic runs in libtlbm's kernels in the
reference's exact operation order (csrc/physics.cuh), so results are
bit-identical to the reference.  Inputs may be numpy arrays (results come back
as numpy) or CUDA tensors (results stay on the device).

Not provided: MRT (collision.py:133-247) -- out of scope for the LBGK hot
path (SURVEY section 8(f)-1 "next").
"""

import enum

import numpy as np
import torch

from . import _native as nat
from .lattice import OPPOSITE, Q


class FluidModel(enum.Enum):
    INCOMPRESSIBLE = "incompressible"
    QUASI_COMPRESSIBLE = "quasi-compressible"


class CollisionModel(enum.Enum):
    LBGK = "lbgk"
    MRT = "mrt"


class DivergenceError(RuntimeError):
    """NaN values or non-positive density (collision.py:38-43)."""

    def __init__(self, message, iteration=None):
        super().__init__(message)
        self.iteration = iteration


def fluid_code(model):
    model = FluidModel(getattr(model, "value", model))
    return nat.QUASI if model is FluidModel.QUASI_COMPRESSIBLE else nat.INCOMPRESSIBLE


def _to_device(a):
    """-> (contiguous CUDA tensor, was_numpy)."""
    if isinstance(a, torch.Tensor):
        dev = nat.require_cuda(a.device.index if a.is_cuda else None)
        return a.to(dev).contiguous(), False
    dev = nat.require_cuda()
    arr = np.ascontiguousarray(a)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    return torch.from_numpy(arr).to(dev), True


def _back(t, as_numpy):
    return t.cpu().numpy() if as_numpy else t


def _flags(dev):
    return torch.zeros(1, dtype=torch.int32, device=dev)


def _raise_if_diverged(flags, what):
    if int(flags.item()) & nat.FLAG_DIVERGED:
        raise DivergenceError(f"non-positive density or NaN in {what}")


def macroscopic(model, f):
    """(rho, u, p) of f with shape (19, ...) (collision.py:75-91); raises
    DivergenceError on rho <= 0 in the quasi-compressible model."""
    ft, as_np = _to_device(f)
    if ft.shape[0] != Q:
        raise ValueError(f"expected 19 populations on axis 0, got {tuple(ft.shape)}")
    rest = tuple(ft.shape[1:])
    n = int(np.prod(rest)) if rest else 1
    rho = torch.empty(n, dtype=ft.dtype, device=ft.device)
    u = torch.empty((3, n), dtype=ft.dtype, device=ft.device)
    p = torch.empty(n, dtype=ft.dtype, device=ft.device)
    flags = _flags(ft.device)
    code = fluid_code(model)
    nat.call("tlbm_macroscopic_canonical", nat.ptr(ft), nat.code_of(ft.dtype), code, n,
             nat.ptr(rho), nat.ptr(u), nat.ptr(p), nat.ptr(flags), nat.stream_ptr(ft.device))
    if code == nat.QUASI:
        _raise_if_diverged(flags, "quasi-compressible flow")
    return (_back(rho.view(rest), as_np), _back(u.view((3,) + rest), as_np),
            _back(p.view(rest), as_np))


def density(f):
    """rho = sum_q f_q in index order (collision.py:55-57)."""
    return macroscopic(FluidModel.INCOMPRESSIBLE, f)[0]


def momentum(f):
    """sum_q c_q f_q in index order (collision.py:60-72)."""
    return macroscopic(FluidModel.INCOMPRESSIBLE, f)[1]


def equilibrium(model, rho, u):
    """(19, ...) equilibria (collision.py:94-121)."""
    rt, as_np = _to_device(rho)
    ut, as_np2 = _to_device(u)
    dt = torch.promote_types(rt.dtype, ut.dtype)
    shape = torch.broadcast_shapes(rt.shape, ut.shape[1:])
    n = int(np.prod(shape)) if len(shape) else 1
    rt = rt.to(dt).expand(shape).contiguous().view(n)
    ut = ut.to(dt).expand((3,) + tuple(shape)).contiguous().view(3, n)
    out = torch.empty((Q, n), dtype=dt, device=rt.device)
    nat.call("tlbm_equilibrium", nat.ptr(rt), nat.ptr(ut), nat.code_of(dt),
             fluid_code(model), n, nat.ptr(out), nat.stream_ptr(rt.device))
    return _back(out.view((Q,) + tuple(shape)), as_np and as_np2)


def collide_lbgk(model, f, tau):
    """f + fl(1/tau) (feq - f) (collision.py:124-130)."""
    ft, as_np = _to_device(f)
    out = ft.clone()
    rest = tuple(ft.shape[1:])
    n = int(np.prod(rest)) if rest else 1
    flags = _flags(ft.device)
    code = fluid_code(model)
    nat.call("tlbm_collide_lbgk", nat.ptr(out), nat.code_of(ft.dtype), code, n,
             float(tau), nat.ptr(flags), nat.stream_ptr(ft.device))
    if code == nat.QUASI:
        _raise_if_diverged(flags, "quasi-compressible flow")
    return _back(out, as_np)


def reflect(f):
    """f_q <- f_opp(q) (collision.py:250-252)."""
    if isinstance(f, torch.Tensor):
        return f[torch.as_tensor(OPPOSITE, device=f.device)]
    ft, _ = _to_device(f)
    return ft[torch.as_tensor(OPPOSITE, device=ft.device)].cpu().numpy()

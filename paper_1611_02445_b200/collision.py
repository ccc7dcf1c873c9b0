"""Node physics API on the GPU: moments, equilibrium, LBGK collision.

Same names, shapes and dtype behaviour as ``tilelbm.collision``
(collision.py:28-130, 250-252); the arithmetic runs in libtlbm's kernels in the
reference's exact operation order (csrc/physics.cuh), so results are
bit-identical to the reference.  Inputs may be numpy arrays (results come back
as numpy) or CUDA tensors (results stay on the device).

MRT (collision.py:133-247): the moment basis, rates and the
19x19 velocity-space operator are host setup in float64 numpy exactly as in
the reference; ``collide_mrt`` and the solver's MRT step apply the operator in
libtlbm (dense 19 x 19 product, coefficients in the kernel-parameter constant
bank, reference accumulation order).
"""

import enum

import numpy as np
import torch

from . import _native as nat
from .lattice import E_VECTORS, OPPOSITE, Q, WEIGHTS  # noqa: F401 (reference namespace)


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


# -- MRT ----------------------------------------------------------------------

def _moment_rows():
    """Orthogonal D3Q19 moment basis, reference row order (collision.py:133-161):
    rho, e, eps, (j, q) per axis, 3pxx, 3pixx, pww, piww, pxy, pyz, pxz, mx,
    my, mz."""
    from .lattice import E_VECTORS
    ex, ey, ez = (E_VECTORS[:, a].astype(np.int64) for a in range(3))
    e2 = ex * ex + ey * ey + ez * ez
    rows = [np.ones(19, dtype=np.int64), 19 * e2 - 30, (21 * e2 * e2 - 53 * e2 + 24) // 2]
    for ea in (ex, ey, ez):
        rows += [ea, (5 * e2 - 9) * ea]
    a_xx, a_ww = 3 * ex * ex - e2, ey * ey - ez * ez
    rows += [a_xx, (3 * e2 - 5) * a_xx, a_ww, (3 * e2 - 5) * a_ww, ex * ey, ey * ez, ex * ez,
             a_ww * ex, (ez * ez - ex * ex) * ey, (ex * ex - ey * ey) * ez]
    return np.stack(rows)


MOMENT_NAMES = ("rho", "e", "eps", "jx", "qx", "jy", "qy", "jz", "qz", "3pxx", "3pixx",
                "pww", "piww", "pxy", "pyz", "pxz", "mx", "my", "mz")
MOMENT_MATRIX = _moment_rows()
CONSERVED_MOMENTS = (0, 3, 5, 7)
STRESS_MOMENTS = (9, 11, 13, 14, 15)


def moment_matrix_inverse():
    """M^T D^-1 by orthogonality (collision.py:179-183)."""
    m = MOMENT_MATRIX.astype(np.float64)
    return m.T / (m * m).sum(axis=1)


def default_mrt_rates(tau):
    """Shear modes at 1/tau, the customary fixed rates elsewhere
    (collision.py:186-203)."""
    if tau <= 0.5:
        raise ValueError(f"relaxation time must exceed 0.5: {tau}")
    s = np.zeros(19)
    s[1], s[2] = 1.19, 1.4
    s[[4, 6, 8]] = 1.2
    s[[10, 12]] = 1.4
    s[list(STRESS_MOMENTS)] = 1.0 / tau
    s[[16, 17, 18]] = 1.98
    return s


def mrt_operator(rates, dtype=np.float64):
    """M^-1 diag(rates) M, float64 then cast (collision.py:206-213)."""
    rates = np.asarray(rates, dtype=np.float64)
    if rates.shape != (19,):
        raise ValueError(f"expected 19 moment rates, got shape {rates.shape}")
    m = MOMENT_MATRIX.astype(np.float64)
    return (moment_matrix_inverse() @ (rates[:, None] * m)).astype(dtype)


def apply_operator(op, delta):
    """A 19x19 operator applied to (19, ...) data as 19 fixed-order row
    accumulations that skip exact-zero coefficients (collision.py:216-231),
    in one kernel (tlbm_apply_operator).  Each term is computed as numpy
    computes ``acc += c * delta[j]`` with ``c`` an element of ``op``: in the
    promoted type of (op, delta), then stored in delta's dtype -- bit-
    identical to the reference for float32 and float64 data."""
    opa = np.asarray(op)
    if opa.shape != (Q, Q):
        raise ValueError(f"operator must be 19x19, got {opa.shape}")
    dt, as_np = _to_device(delta)
    if dt.shape[0] != Q:
        raise ValueError(f"expected (19, ...) data, got {tuple(dt.shape)}")
    wide = int(opa.dtype == np.float64 and dt.dtype == torch.float32)
    op64 = np.ascontiguousarray(opa, dtype=np.float64)
    src = dt.contiguous()
    out = torch.empty_like(src)
    n = src.numel() // Q
    nat.call("tlbm_apply_operator", nat.ptr(src), nat.ptr(out), nat.code_of(src.dtype), n,
             op64.ctypes.data, wide, nat.stream_ptr(src.device))
    return _back(out, as_np)


def collide_mrt(model, f, rates=None, operator=None):
    """f + M^-1 S M (feq - f) (collision.py:234-247) on the GPU.  With
    ``rates`` the operator is built in float64 and rounded to f's dtype, as
    the reference does; an explicit float64 ``operator`` on float32 data is
    applied the way NumPy promotes it (each term in float64, rounded into
    the float32 accumulator)."""
    ft, as_np = _to_device(f)
    if operator is None:
        if rates is None:
            raise ValueError("either moment rates or a precomputed operator is required")
        operator = mrt_operator(rates, dtype=np.float64)
        wide = False
    else:
        wide = np.asarray(operator).dtype == np.float64 and ft.dtype == torch.float32
    op = np.ascontiguousarray(np.asarray(operator, dtype=np.float64))
    out = ft.clone()
    rest = tuple(ft.shape[1:])
    n = int(np.prod(rest)) if rest else 1
    flags = _flags(ft.device)
    code = fluid_code(model)
    if wide:
        nat.call("tlbm_collide_mrt_wide", nat.ptr(out), code, n, op.ctypes.data, nat.ptr(flags),
                 nat.stream_ptr(ft.device))
    else:
        nat.call("tlbm_collide_mrt", nat.ptr(out), nat.code_of(ft.dtype), code, n,
                 op.ctypes.data, nat.ptr(flags), nat.stream_ptr(ft.device))
    if code == nat.QUASI:
        _raise_if_diverged(flags, "quasi-compressible flow")
    return _back(out, as_np)

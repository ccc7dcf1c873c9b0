"""Dense-grid restatement of one LBGK step.

The reference has no step function; this composes the
pinned numerics (oracle/numerics.py) with the step contract of
boundaries.py:1-28, SPEC.md:388-401,421-425 and PAPER.md:763-788:

R2 gather   g_q(n) = f_q(n - e_q) if n - e_q is in the domain (or wrapped on a
            periodic axis) and non-solid, else f_opp(q)(n)  (halfway BB fill)
R3 dispatch FLUID -> collide; BB_WALL -> g[opp] (collision.py:250-252);
            VELOCITY_INLET / PRESSURE_OUTLET -> Zou-He on the node's unique
            face (boundaries.py:95-195), then collide
R4 collide  collide_lbgk (collision.py:124-130)
R5 store    into the other copy; SOLID nodes are never written
"""

import numpy as np

from . import numerics as nm

SOLID, FLUID, BB_WALL, INLET, OUTLET = 0, 1, 2, 3, 4


def face_ids(types, periodic=(False, False, False)):
    """Per node: 2*axis + (0 low | 1 high) for inlet/outlet nodes, -1 else.

    Mirrors classify_boundary_faces (boundaries.py:95-129): an inlet/outlet
    node must lie on exactly one domain face (faces of periodic axes do not
    count -- extension) or ValueError is raised.
    """
    dims = types.shape
    io = (types == INLET) | (types == OUTLET)
    out = np.full(dims, -1, dtype=np.int8)
    ids = np.flatnonzero(io)
    if ids.size == 0:
        return out
    c = np.stack(np.unravel_index(ids, dims), axis=1)
    lo = c == 0
    hi = c == np.asarray(dims) - 1
    for a in range(3):
        if periodic[a]:
            lo[:, a] = False
            hi[:, a] = False
    cnt = lo.sum(1) + hi.sum(1)
    if np.any(cnt != 1):
        x, y, z = c[np.argmax(cnt != 1)]
        raise ValueError(f"inlet/outlet node ({x}, {y}, {z}) does not lie on "
                         "exactly one axis-aligned domain face")
    face = np.where(lo.any(1), 2 * np.argmax(lo, 1), 2 * np.argmax(hi, 1) + 1)
    out.ravel()[ids] = face
    return out


def _pull(arr, ok, e, periodic):
    """Return (arr[n - e], ok[n - e]) with off-domain -> (0, False)."""
    val, valid = arr, ok
    for a in range(3):
        s = int(e[a])
        if s == 0:
            continue
        if periodic[a]:
            val = np.roll(val, s, axis=a)
            valid = np.roll(valid, s, axis=a)
            continue
        v2 = np.zeros_like(val)
        k2 = np.zeros_like(valid)
        dst = [slice(None)] * 3
        src = [slice(None)] * 3
        dst[a] = slice(1, None) if s > 0 else slice(None, -1)
        src[a] = slice(None, -1) if s > 0 else slice(1, None)
        v2[tuple(dst)] = val[tuple(src)]
        k2[tuple(dst)] = valid[tuple(src)]
        val, valid = v2, k2
    return val, valid


def gather(f, types, periodic=(False, False, False)):
    ok = types != SOLID
    g = np.empty_like(f)
    g[0] = f[0]
    for q in range(1, 19):
        v, k = _pull(f[q], ok, nm.E[q], periodic)
        g[q] = np.where(k, v, f[nm.OPP[q]])
    return g


def step(f, types, model, tau, inlet_velocity=(0.0, 0.0, 0.0),
         outlet_density=1.0, periodic=(False, False, False), faces=None,
         iteration=None, mrt_operator=None):
    """One step on dense f of shape (19, nx, ny, nz); returns the new copy.
    ``mrt_operator`` (19x19) selects MRT collision (collision.py:234-247)."""
    if faces is None:
        faces = face_ids(types, periodic)
    if mrt_operator is None:
        collide = lambda g: nm.collide_lbgk(model, g, tau)  # noqa: E731
    else:
        collide = lambda g: nm.collide_mrt(model, g, operator=mrt_operator)  # noqa: E731
    g = gather(f, types, periodic)
    new = f.copy()
    fl = types == FLUID
    try:
        new[:, fl] = collide(g[:, fl])
        bb = types == BB_WALL
        new[:, bb] = g[nm.OPP][:, bb]
        for fid in range(6):
            c = nm.FACES[(fid // 2, 1 if fid % 2 == 0 else -1)]
            for tag in (INLET, OUTLET):
                m = (types == tag) & (faces == fid)
                if not m.any():
                    continue
                sub = g[:, m].copy()
                if tag == INLET:
                    nm.zou_he_velocity(sub, c, inlet_velocity, model)
                else:
                    nm.zou_he_pressure(sub, c, outlet_density, model)
                new[:, m] = collide(sub)
    except nm.OracleDivergence as exc:
        raise nm.OracleDivergence(str(exc), iteration) from None
    ns = types != SOLID
    if np.isnan(nm.density(new[:, ns])).any():
        raise nm.OracleDivergence("NaN in distributions", iteration)
    return new


def init_equilibrium(types_shape, model, dtype, rho=1.0, u=(0.0, 0.0, 0.0)):
    """f = equilibrium(rho, u) everywhere."""
    dt = np.dtype(dtype)
    r = np.full(types_shape, rho, dtype=dt)
    uu = np.stack([np.full(types_shape, c, dtype=dt) for c in u])
    return nm.equilibrium(model, r, uu)


def run(f, types, model, tau, steps, **kw):
    faces = face_ids(types, kw.get("periodic", (False, False, False)))
    for i in range(steps):
        f = step(f, types, model, tau, faces=faces, iteration=i, **kw)
    return f


def to_canonical(f_dense, non_empty, fill, a=4):
    """Dense (19, nx, ny, nz) -> canonical (19, t_n, 64); padding slots take
    ``fill[q]`` (the init value, since padding is never written)."""
    q, nx, ny, nz = f_dense.shape
    pd = [(-(-n // a)) * a for n in (nx, ny, nz)]
    pad = np.empty((q,) + tuple(pd), dtype=f_dense.dtype)
    pad[:] = np.asarray(fill, dtype=f_dense.dtype).reshape(q, 1, 1, 1)
    pad[:, :nx, :ny, :nz] = f_dense
    s = np.arange(64)
    x = non_empty[:, 0:1] + (s & 3)
    y = non_empty[:, 1:2] + ((s >> 2) & 3)
    z = non_empty[:, 2:3] + (s >> 4)
    return pad[:, x, y, z]


def from_canonical(canon, non_empty, dims):
    """Canonical (19, t_n, 64) -> dense (19, nx, ny, nz) (absent tiles = 0)."""
    nx, ny, nz = dims
    pd = [(-(-n // 4)) * 4 for n in dims]
    out = np.zeros((canon.shape[0],) + tuple(pd), dtype=canon.dtype)
    s = np.arange(64)
    x = non_empty[:, 0:1] + (s & 3)
    y = non_empty[:, 1:2] + ((s >> 2) & 3)
    z = non_empty[:, 2:3] + (s >> 4)
    out[:, x, y, z] = canon
    return out[:, :nx, :ny, :nz]

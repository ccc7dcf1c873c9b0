"""Reference arithmetic restated in numpy, operation-for-operation.

Every function keeps the dtype of its inputs and evaluates in the exact order
the reference does, so results are bit-identical to ``tilelbm`` (checked by
tests/test_oracle.py against the reference functions and golden vectors).

Order rules:
  rho   = ((f0 + f1) + f2) + ... + f18                 collision.py:46-57
  j_a   = ((0 (+/-) f_q1) (+/-) f_q2) ...  in q order  collision.py:60-72
  cu    = ((0 (+/-) ux) (+/-) uy) (+/-) uz             collision.py:108-114
  br    = ((3 cu) + ((4.5 cu) cu)) - (1.5 usq)         collision.py:116
  feq   = w (rho + br) | w (rho (1 + br))              collision.py:117-120
  post  = f + fl(1/tau) (feq - f)                      collision.py:124-130
  Zou-He sums in the closure's tuple order            boundaries.py:132-195
"""

import numpy as np

E = np.array([(0, 0, 0), (1, 0, 0), (0, 1, 0), (-1, 0, 0), (0, -1, 0),
              (0, 0, 1), (0, 0, -1), (1, 1, 0), (-1, 1, 0), (1, -1, 0),
              (-1, -1, 0), (0, 1, 1), (0, 1, -1), (0, -1, 1), (0, -1, -1),
              (1, 0, 1), (1, 0, -1), (-1, 0, 1), (-1, 0, -1)], dtype=np.int64)
OPP = np.array([0, 3, 4, 1, 2, 6, 5, 10, 9, 8, 7, 14, 13, 12, 11, 18, 17, 16,
                15], dtype=np.int64)
W = np.array([1 / 3] + [1 / 18] * 6 + [1 / 36] * 12)

INCOMPRESSIBLE = "incompressible"
QUASI_COMPRESSIBLE = "quasi-compressible"


class OracleDivergence(RuntimeError):
    def __init__(self, message, iteration=None):
        super().__init__(message)
        self.iteration = iteration


def _model(model):
    """Accept the reference/product enum or its string value."""
    v = getattr(model, "value", model)
    if v not in (INCOMPRESSIBLE, QUASI_COMPRESSIBLE):
        raise ValueError(f"unknown fluid model {model!r}")
    return v


def density(f):
    acc = f[0].copy()
    for q in range(1, 19):
        acc += f[q]
    return acc


def momentum(f):
    out = []
    for a in range(3):
        acc = np.zeros_like(f[0])
        for q in range(19):
            s = E[q, a]
            if s > 0:
                acc += f[q]
            elif s < 0:
                acc -= f[q]
        out.append(acc)
    return np.stack(out)


def macroscopic(model, f):
    f = np.asarray(f)
    rho = density(f)
    j = momentum(f)
    if _model(model) == QUASI_COMPRESSIBLE:
        if np.any(rho <= 0):
            raise OracleDivergence("non-positive density in quasi-compressible flow")
        u = j / rho
    else:
        u = j
    return rho, u, rho / np.asarray(3.0, dtype=rho.dtype)


def equilibrium(model, rho, u):
    rho = np.asarray(rho)
    u = np.asarray(u)
    dt = np.result_type(rho, u)
    T = dt.type
    ux, uy, uz = u[0], u[1], u[2]
    usq = ux * ux + uy * uy + uz * uz
    quasi = _model(model) == QUASI_COMPRESSIBLE
    out = np.empty((19,) + np.broadcast_shapes(rho.shape, usq.shape), dtype=dt)
    comps = (ux, uy, uz)
    for q in range(19):
        cu = np.zeros_like(usq)
        for a in range(3):
            if E[q, a] > 0:
                cu += comps[a]
            elif E[q, a] < 0:
                cu += -comps[a]
        br = T(3.0) * cu + T(4.5) * cu * cu - T(1.5) * usq
        w = T(W[q])
        out[q] = w * (rho * (T(1.0) + br)) if quasi else w * (rho + br)
    return out


def collide_lbgk(model, f, tau):
    f = np.asarray(f)
    rho, u, _ = macroscopic(model, f)
    feq = equilibrium(model, rho, u)
    return f + f.dtype.type(1.0 / tau) * (feq - f)


def reflect(f):
    return np.asarray(f)[OPP]


# -- Zou-He face closures (boundaries.py:39-92) -----------------------------

def face_closure(axis, sign):
    """Index sets of one face: dict with unknown axis pair, diagonals
    (q, opp, tau, sigma), k0 (c.n = 0), km (c.n = -1) and tangential sets."""
    n = np.zeros(3, dtype=np.int64)
    n[axis] = sign
    cn = E @ n
    k0 = tuple(int(q) for q in range(19) if cn[q] == 0)
    km = tuple(int(q) for q in range(19) if cn[q] == -1)
    diag = []
    ax_dir = None
    for q in range(19):
        if cn[q] != 1:
            continue
        side = [a for a in range(3) if a != axis and E[q, a] != 0]
        if side:
            diag.append((q, int(OPP[q]), side[0], int(E[q, side[0]])))
        else:
            ax_dir = q
    tang = {}
    for tau in range(3):
        if tau == axis:
            continue
        tang[tau] = (tuple(q for q in k0 if E[q, tau] == 1),
                     tuple(q for q in k0 if E[q, tau] == -1))
    return {"axis": axis, "sign": sign, "t": ax_dir, "t_opp": int(OPP[ax_dir]),
            "diagonals": tuple(diag), "k0": k0, "km": km, "tangential": tang}


FACES = {(a, s): face_closure(a, s) for a in range(3) for s in (1, -1)}


def _osum(g, dirs):
    acc = g[dirs[0]].copy()
    for q in dirs[1:]:
        acc += g[q]
    return acc


def _close(g, c, j):
    T = g.dtype.type
    jn = T(c["sign"]) * j[c["axis"]]
    g[c["t"]] = g[c["t_opp"]] + T(1.0 / 3.0) * jn
    ntau = {}
    for tau, (plus, minus) in c["tangential"].items():
        ntau[tau] = T(0.5) * (_osum(g, plus) - _osum(g, minus)) - T(1.0 / 3.0) * j[tau]
    for q, qo, tau, sg in c["diagonals"]:
        s = T(sg)
        g[q] = g[qo] + T(1.0 / 6.0) * (jn + s * j[tau]) - s * ntau[tau]


def zou_he_velocity(g, c, u, model):
    T = g.dtype.type
    u = np.asarray(u, dtype=g.dtype)
    un = T(c["sign"]) * u[c["axis"]]
    k0 = _osum(g, c["k0"])
    km = _osum(g, c["km"])
    if _model(model) == QUASI_COMPRESSIBLE:
        rho = (k0 + T(2.0) * km) / (T(1.0) - un)
        j = u[:, None] * rho
    else:
        rho = k0 + T(2.0) * km + un
        j = np.broadcast_to(u[:, None], (3, g.shape[1])).copy()
    _close(g, c, j)
    return rho


def zou_he_pressure(g, c, rho0, model):
    T = g.dtype.type
    rho0 = T(rho0)
    k0 = _osum(g, c["k0"])
    km = _osum(g, c["km"])
    jn = rho0 - (k0 + T(2.0) * km)
    j = np.zeros((3, g.shape[1]), dtype=g.dtype)
    j[c["axis"]] = T(c["sign"]) * jn
    _close(g, c, j)
    return jn


# -- MRT (collision.py:133-247) ------------------------------------------------

def moment_rows():
    """Orthogonal D3Q19 moment basis in the reference's row order
    (collision.py:133-161)."""
    ex, ey, ez = E[:, 0], E[:, 1], E[:, 2]
    e2 = ex * ex + ey * ey + ez * ez
    r = [np.ones(19, dtype=np.int64), 19 * e2 - 30, (21 * e2 * e2 - 53 * e2 + 24) // 2]
    for ea in (ex, ey, ez):
        r += [ea, (5 * e2 - 9) * ea]
    r += [3 * ex * ex - e2, (3 * e2 - 5) * (3 * ex * ex - e2), ey * ey - ez * ez,
          (3 * e2 - 5) * (ey * ey - ez * ez), ex * ey, ey * ez, ex * ez,
          (ey * ey - ez * ez) * ex, (ez * ez - ex * ex) * ey, (ex * ex - ey * ey) * ez]
    return np.stack(r)


MOMENTS = moment_rows()
STRESS = (9, 11, 13, 14, 15)


def default_mrt_rates(tau):
    """collision.py:186-203."""
    if tau <= 0.5:
        raise ValueError(f"relaxation time must exceed 0.5: {tau}")
    s = np.zeros(19)
    s[1], s[2] = 1.19, 1.4
    s[4] = s[6] = s[8] = 1.2
    s[10] = s[12] = 1.4
    for i in STRESS:
        s[i] = 1.0 / tau
    s[16] = s[17] = s[18] = 1.98
    return s


def mrt_operator(rates, dtype=np.float64):
    """M^-1 diag(s) M in float64 via numpy matmul, cast (collision.py:206-213)."""
    m = MOMENTS.astype(np.float64)
    inv = m.T / (m * m).sum(axis=1)
    rates = np.asarray(rates, dtype=np.float64)
    return (inv @ (rates[:, None] * m)).astype(dtype)


def apply_operator(op, delta):
    """Fixed-order accumulation skipping zero coefficients (collision.py:216-231)."""
    out = np.empty_like(delta)
    for i in range(19):
        acc = np.zeros_like(delta[0])
        for j in range(19):
            c = op[i][j]
            if c != 0.0:
                acc += c * delta[j]
        out[i] = acc
    return out


def collide_mrt(model, f, rates=None, operator=None):
    f = np.asarray(f)
    if operator is None:
        if rates is None:
            raise ValueError("either moment rates or a precomputed operator is required")
        operator = mrt_operator(rates, dtype=f.dtype)
    rho, u, _ = macroscopic(model, f)
    feq = equilibrium(model, rho, u)
    return f + apply_operator(operator, feq - f)

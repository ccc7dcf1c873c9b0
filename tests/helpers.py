"""Shared test helpers."""

import numpy as np


def random_geometry(rng, shape, periodic=(False, False, False), io_axis=2):
    """Mixed SOLID/FLUID/BB interior with inlet (low face) / outlet (high
    face) on the faces normal to ``io_axis``; the other non-periodic faces
    and the rim of the inlet/outlet faces are bounce-back."""
    t = rng.choice([0, 1, 1, 1, 2], size=shape).astype(np.uint8)
    for a in range(3):
        if periodic[a] or a == io_axis:
            continue
        sl = [slice(None)] * 3
        for idx in (0, shape[a] - 1):
            sl[a] = idx
            face = t[tuple(sl)]
            face[face != 0] = 2
    if io_axis is not None and not periodic[io_axis]:
        lo = np.moveaxis(t, io_axis, 0)[0]
        hi = np.moveaxis(t, io_axis, 0)[-1]
        inner = np.zeros(lo.shape, dtype=bool)
        inner[1:-1, 1:-1] = True
        lo[(lo == 1) & inner] = 3
        hi[(hi == 1) & inner] = 4
        lo[(lo == 1) & ~inner] = 2
        hi[(hi == 1) & ~inner] = 2
    return t

"""Shared test helpers."""

import numpy as np


def random_geometry(rng, shape, periodic=(False, False, False)):
    """Mixed SOLID/FLUID/BB interior with inlet/outlet on the z faces."""
    t = rng.choice([0, 1, 1, 1, 2], size=shape).astype(np.uint8)
    for a in range(2):
        if periodic[a]:
            continue
        sl = [slice(None)] * 3
        for idx in (0, shape[a] - 1):
            sl[a] = idx
            face = t[tuple(sl)]
            face[face != 0] = 2
    if not periodic[2]:
        lo, hi = t[:, :, 0], t[:, :, -1]
        inner = np.zeros(lo.shape, dtype=bool)
        inner[1:-1, 1:-1] = True
        lo[(lo == 1) & inner] = 3
        hi[(hi == 1) & inner] = 4
        lo[(lo == 1) & ~inner] = 2
        hi[(hi == 1) & ~inner] = 2
    return t

"""B200-native tiled sparse-geometry D3Q19 lattice-Boltzmann step
(arXiv 1611.02445), drop-in for the ``tilelbm`` reference's Python API.

Modules mirror the reference: lattice, geometry, tiling, layout, collision,
boundaries, txmodel, plus the solver the reference only specifies
(SPEC.md:330-433).  All compute runs in libtlbm.so (sm_100a CUDA, C ABI in
include/tlbm.h) through ctypes; there is no CPU fallback.
"""

from . import lattice, geometry  # noqa: F401  (pure host modules)

__all__ = ["lattice", "geometry", "tiling", "layout", "collision", "boundaries",
           "txmodel", "solver"]


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)

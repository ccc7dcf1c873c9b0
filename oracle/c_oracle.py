"""ctypes wrapper of the C oracle (oracle/tlbm_oracle.c) -- TEST INFRASTRUCTURE.

``run_dense`` advances a dense (19, nx, ny, nz) field ``steps`` steps with the
same rules and arithmetic as oracle/dense.py, multithreaded with OpenMP.
"""

import ctypes
import os
import subprocess

import numpy as np

from .dense import face_ids

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")


class _Params(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("periodic", ctypes.c_int * 3), ("quasi", ctypes.c_int),
                ("tau", ctypes.c_double), ("inlet_u", ctypes.c_double * 3),
                ("outlet_rho", ctypes.c_double), ("u_guard", ctypes.c_double),
                ("nthreads", ctypes.c_int), ("mrt_op", ctypes.c_void_p)]


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        for sfx in ("f64", "f32"):
            fn = getattr(_lib, f"oracle_run_{sfx}")
            fn.restype = ctypes.c_int
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.POINTER(_Params), ctypes.c_int,
                           ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
    return _lib


def _model_is_quasi(model):
    return getattr(model, "value", model) == "quasi-compressible"


class DenseOracle:
    """Holds the two dense copies and the geometry of one oracle run."""

    def __init__(self, types, model, tau, inlet_velocity=(0.0, 0.0, 0.0),
                 outlet_density=1.0, periodic=(False, False, False), f0=None,
                 dtype=np.float64, nthreads=0, u_guard=0.0, mrt_operator=None):
        self.types = np.ascontiguousarray(types, dtype=np.uint8)
        self.faces = np.ascontiguousarray(face_ids(self.types, periodic))
        self.dtype = np.dtype(dtype)
        if f0 is None:
            raise ValueError("initial dense field f0 is required")
        self.a = np.ascontiguousarray(f0, dtype=self.dtype).copy()
        self.b = self.a.copy()
        self.which = 0
        p = _Params()
        p.nx, p.ny, p.nz = self.types.shape
        p.periodic[:] = [int(bool(v)) for v in periodic]
        p.quasi = int(_model_is_quasi(model))
        p.tau = float(tau)
        p.inlet_u[:] = [float(v) for v in inlet_velocity]
        p.outlet_rho = float(outlet_density)
        p.u_guard = float(u_guard)
        p.nthreads = int(nthreads)
        self.mrt_op = None
        if mrt_operator is not None:
            self.mrt_op = np.ascontiguousarray(mrt_operator, dtype=self.dtype)
            p.mrt_op = self.mrt_op.ctypes.data
        self.params = p
        self.last_status = 0
        self.failed_step = -1

    @property
    def f(self):
        return self.a if self.which == 0 else self.b

    def run(self, steps):
        fn = lib().oracle_run_f64 if self.dtype == np.float64 else lib().oracle_run_f32
        cur, oth = (self.a, self.b) if self.which == 0 else (self.b, self.a)
        which = ctypes.c_int(0)
        failed = ctypes.c_int(-1)
        st = fn(cur.ctypes.data, oth.ctypes.data, self.types.ctypes.data,
                self.faces.ctypes.data, ctypes.byref(self.params), int(steps),
                ctypes.byref(which), ctypes.byref(failed))
        # which is relative to (cur, oth)
        if which.value == 1:
            self.which ^= 1
        self.last_status = st
        self.failed_step = failed.value
        return st

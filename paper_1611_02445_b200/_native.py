"""ctypes binding of libtlbm.so (include/tlbm.h).

The library is the product: there is no Python/CPU fallback.  If it is
missing or fails to load, every entry point raises immediately.
"""

import ctypes
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TLBM_LIB") or os.path.join(HERE, "lib", "libtlbm.so")
ABI_VERSION = 3

F64, F32 = 0, 1
INCOMPRESSIBLE, QUASI = 0, 1
TABLE_XYZ, TABLE_OPTIMIZED, TABLE_B200 = 0, 1, 2
FULL, PROPAGATION_ONLY, READ_WRITE_ONLY = 0, 1, 2
LBGK, MRT = 0, 1
ARITH_REFERENCE, ARITH_FMA = 0, 1
FLAG_DIVERGED, FLAG_GUARD = 1, 2

c_int, c_i64, c_dbl, c_vp = ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
c_size = ctypes.c_size_t


class StepArgs(ctypes.Structure):
    _fields_ = [("dtype", c_int), ("fluid", c_int), ("table", c_int), ("variant", c_int),
                ("t_n", c_i64), ("tile_begin", c_i64), ("tile_end", c_i64),
                ("f_src", c_vp), ("f_dst", c_vp), ("nbr", c_vp), ("meta", c_vp),
                ("tau", c_dbl), ("inlet_u", c_dbl * 3), ("outlet_rho", c_dbl),
                ("u_guard", c_dbl), ("flags", c_vp), ("rel32", c_int),
                ("halo_up", c_vp), ("halo_up_begin", c_i64), ("halo_up_end", c_i64),
                ("halo_down", c_vp), ("halo_down_begin", c_i64), ("halo_down_end", c_i64),
                ("collision", c_int), ("mrt_op", c_vp), ("arith", c_int),
                ("iter_counter", c_vp), ("iter_add", c_i64), ("ring_len", c_int),
                ("cbase", c_vp), ("cnf", c_vp), ("crank", c_vp), ("order", c_vp),
                ("halo_up_cbase", c_vp), ("halo_down_cbase", c_vp),
                ("node_meta", c_vp), ("node_rec", c_vp), ("unit_tile", c_vp),
                ("entries", c_vp), ("node_begin", c_i64), ("node_end", c_i64)]


_PROTOS = {
    "tlbm_abi_version": (c_int, []),
    "tlbm_last_error": (ctypes.c_char_p, []),
    "tlbm_set_device": (c_int, [c_int]),
    "tlbm_set_l2_fetch_granularity": (c_int, [c_int]),
    "tlbm_get_l2_fetch_granularity": (c_int, [ctypes.POINTER(c_int)]),
    "tlbm_lattice_tables": (c_int, [c_int, c_vp, c_vp, c_vp, c_vp]),
    "tlbm_tiling_scratch_bytes": (c_size, [c_int, c_int, c_int]),
    "tlbm_tile_map": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_vp,
                              ctypes.POINTER(c_i64), c_vp]),
    "tlbm_tile_list": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_i64, c_vp]),
    "tlbm_tile_neighbors": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_i64, c_int,
                                    c_vp, c_vp]),
    "tlbm_node_meta": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_vp, c_i64, c_vp,
                               c_vp, c_vp]),
    "tlbm_tile_counts": (c_int, [c_vp, c_i64, c_vp, c_vp]),
    "tlbm_init_equilibrium": (c_int, [c_vp, c_int, c_int, c_int, c_i64, c_dbl, c_dbl,
                                      c_dbl, c_dbl, c_vp]),
    "tlbm_init_from_macroscopic": (c_int, [c_vp, c_int, c_int, c_int, c_i64, c_vp,
                                           c_vp, c_vp]),
    "tlbm_to_canonical": (c_int, [c_vp, c_int, c_int, c_i64, c_vp, c_vp]),
    "tlbm_from_canonical": (c_int, [c_vp, c_int, c_int, c_i64, c_vp, c_vp]),
    "tlbm_macroscopic": (c_int, [c_vp, c_int, c_int, c_int, c_i64, c_vp, c_vp, c_vp,
                                 c_vp, c_vp]),
    "tlbm_macroscopic_canonical": (c_int, [c_vp, c_int, c_int, c_i64, c_vp, c_vp,
                                           c_vp, c_vp, c_vp]),
    "tlbm_equilibrium": (c_int, [c_vp, c_vp, c_int, c_int, c_i64, c_vp, c_vp]),
    "tlbm_collide_lbgk": (c_int, [c_vp, c_int, c_int, c_i64, c_dbl, c_vp, c_vp]),
    "tlbm_collide_mrt": (c_int, [c_vp, c_int, c_int, c_i64, c_vp, c_vp, c_vp]),
    "tlbm_collide_mrt_wide": (c_int, [c_vp, c_int, c_i64, c_vp, c_vp, c_vp]),
    "tlbm_apply_operator": (c_int, [c_vp, c_vp, c_int, c_i64, c_vp, c_int, c_vp]),
    "tlbm_zou_he": (c_int, [c_vp, c_int, c_int, c_int, c_int, c_i64, c_dbl, c_dbl,
                            c_dbl, c_dbl, c_vp, c_vp]),
    "tlbm_halo": (c_int, [c_vp, c_int, c_int, c_i64, c_i64, c_int, c_int, c_vp, c_vp]),
    "tlbm_step": (c_int, [ctypes.POINTER(StepArgs), c_vp]),
    "tlbm_advance_counter": (c_int, [c_vp, c_i64, c_vp]),
    "tlbm_vessel_tree": (c_int, [c_vp, c_vp, c_int, c_int, c_int, c_int, c_int, c_vp, c_vp,
                                 c_vp]),
    "tlbm_compact_ranks": (c_int, [c_vp, c_i64, c_vp, c_vp]),
    "tlbm_compact_nodes": (c_int, [c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                   c_vp, c_vp, c_vp]),
    "tlbm_sphere_cover": (c_int, [c_vp, c_i64, c_i64, c_int, c_dbl, c_vp, c_vp]),
    "tlbm_halo_compact": (c_int, [c_vp, c_int, c_i64, c_i64, c_int, c_int, c_vp, c_vp, c_vp,
                                  c_vp, c_vp]),
    "tlbm_compact_convert": (c_int, [c_vp, c_vp, c_int, c_int, c_i64, c_vp, c_vp, c_vp, c_int,
                                     c_vp]),
    "tlbm_ipc_export": (c_int, [c_vp, c_vp, ctypes.POINTER(ctypes.c_uint64)]),
    "tlbm_ipc_import": (c_int, [c_vp, ctypes.c_uint64, ctypes.POINTER(c_vp)]),
    "tlbm_ipc_close": (c_int, [c_vp]),
    "tlbm_peer_wait": (c_int, [c_vp, c_int, ctypes.c_uint64, ctypes.c_uint64, c_vp, c_vp]),
    "tlbm_peer_signal": (c_int, [c_vp, c_vp, ctypes.c_uint64, c_vp]),
}

EXPORTED = tuple(_PROTOS)

_lib = None


def load():
    """Load libtlbm.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"libtlbm.so not found at {LIB_PATH}; build it with `make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` -- there is no "
            "CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.tlbm_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libtlbm ABI {lib.tlbm_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc):
    if rc != 0:
        msg = load().tlbm_last_error().decode(errors="replace")
        raise RuntimeError(f"libtlbm error {rc}: {msg}")


def call(name, *args):
    check(getattr(load(), name)(*args))


def require_cuda(device=None):
    """Select the CUDA device for the next calls; raise without a GPU."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1611_02445_b200 needs a CUDA device (no CPU fallback)")
    if isinstance(device, torch.device):
        if device.type != "cuda":
            raise RuntimeError(f"not a CUDA device: {device}")
        device = device.index
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    check(load().tlbm_set_device(dev.index))
    return dev


def stream_ptr(device=None):
    return c_vp(torch.cuda.current_stream(device).cuda_stream)


def ptr(t):
    return c_vp(t.data_ptr()) if t is not None else c_vp(0)


def torch_dtype(code):
    return torch.float64 if code == F64 else torch.float32


def code_of(dtype):
    """Map numpy/torch/str dtype to the ABI code."""
    if isinstance(dtype, torch.dtype):
        if dtype == torch.float64:
            return F64
        if dtype == torch.float32:
            return F32
    elif dtype in ("f64", "float64"):
        return F64
    elif dtype in ("f32", "float32"):
        return F32
    else:
        nd = np.dtype(dtype)
        if nd == np.float64:
            return F64
        if nd == np.float32:
            return F32
    raise ValueError(f"unsupported dtype {dtype!r}: only float64 and float32")


def lattice_tables(table):
    e = np.zeros((19, 3), dtype=np.int32)
    o = np.zeros(19, dtype=np.int32)
    w = np.zeros(19, dtype=np.float64)
    p = np.zeros((19, 64), dtype=np.int32)
    check(load().tlbm_lattice_tables(int(table), e.ctypes.data, o.ctypes.data,
                                     w.ctypes.data, p.ctypes.data))
    return e, o, w, p

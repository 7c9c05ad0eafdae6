"""ctypes binding of libpgcp_b200.so (include/pgcp_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every compute entry point raises.
"""

import ctypes
import os
import threading

from .errors import MeshError, PartitionError, SolveError, ValidationError, WeldError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpgcp_b200.so")

OK = 0
E_INVALID, E_MESH, E_PARTITION, E_SOLVE, E_NOCONV, E_WELD, E_CUDA, E_VALIDATION = range(1, 9)

ARR_FACE_COMP, ARR_VERT_OFF, ARR_VMAP, ARR_LOOP_OFF, ARR_LOOP, ARR_L_ROWPTR, ARR_L_COL, \
    ARR_L_VAL, ARR_W3, ARR_PINS, ARR_CYCLES = range(11)

INFO_K, INFO_SUM_N, INFO_SUM_NB, INFO_NNZ_L, INFO_PARENT_CHI, INFO_PARENT_LOOPS, INFO_N, \
    INFO_M, INFO_BAD_COMP = range(9)
INFO_COUNT = 16
BATCH_NO_CUTS = 1
BATCH_VALIDATE_ONLY = 2


class SolveOpts(ctypes.Structure):
    _fields_ = [("rtol", ctypes.c_double), ("contract_tol", ctypes.c_double),
                ("maxit", ctypes.c_int32), ("cluster", ctypes.c_int32),
                ("solver", ctypes.c_int32), ("reserved", ctypes.c_int32)]


SOLVERS = {"default": 0, "direct": 1, "pcg": 2}


class SolveStat(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("status", ctypes.c_int32), ("relres", ctypes.c_double),
                ("true_res", ctypes.c_double), ("bnorm", ctypes.c_double), ("xnorm", ctypes.c_double)]


# int (*pgcp_reduce_fn)(void* buf, int64_t count, int dtype, int op, void* user, void* stream)
REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                             ctypes.c_void_p, ctypes.c_void_p)


class Rec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("flags", ctypes.c_int32), ("p", ctypes.c_double * 16)]


_lock = threading.Lock()
_lib = None

_VP = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_U32 = ctypes.c_uint32
_D = ctypes.c_double
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PD = ctypes.POINTER(ctypes.c_double)

_SIGS = {
    "pgcp_abi_version": ([], ctypes.c_int),
    "pgcp_last_error": ([], ctypes.c_char_p),
    "pgcp_batch_create": ([_VP, _VP, _I64, _I64, _VP, _I64, _U32, _VP, ctypes.POINTER(_VP)], ctypes.c_int),
    "pgcp_batch_destroy": ([_VP], ctypes.c_int),
    "pgcp_batch_release_solvers": ([_VP, ctypes.c_int], ctypes.c_int),
    "pgcp_batch_create_from": ([_VP, _VP, _I64, _U32, _VP, ctypes.POINTER(_VP)], ctypes.c_int),
    "pgcp_batch_info": ([_VP, _PI64, ctypes.c_int], ctypes.c_int),
    "pgcp_batch_array": ([_VP, ctypes.c_int, ctypes.POINTER(_VP), _PI64], ctypes.c_int),
    "pgcp_batch_local_faces": ([_VP, _PI64, _VP, _VP], ctypes.c_int),
    "pgcp_batch_laplacian": ([_VP, _PI64, _VP], ctypes.c_int),
    "pgcp_batch_default_pins": ([_VP, _VP], ctypes.c_int),
    "pgcp_batch_flatten": ([_VP, _VP, _I32, _VP, _PD, ctypes.POINTER(SolveOpts), _VP,
                            ctypes.POINTER(SolveStat), _VP], ctypes.c_int),
    "pgcp_batch_harmonic": ([_VP, _VP, _I32, _VP, _VP, _I64, ctypes.POINTER(SolveOpts), _VP,
                             ctypes.POINTER(SolveStat), _VP], ctypes.c_int),
    "pgcp_batch_harmonic_prepare": ([_VP, _VP, _I32, _VP, _I64, ctypes.POINTER(SolveOpts), _VP], ctypes.c_int),
    "pgcp_batch_harmonic_solve": ([_VP, _VP, _I64, ctypes.POINTER(SolveOpts), _VP, ctypes.POINTER(SolveStat), _VP],
                                  ctypes.c_int),
    "pgcp_batch_export_system": ([_VP, ctypes.c_int, _I32, _PI64, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "pgcp_batch_conformal_energy": ([_VP, _VP, _PD, _VP], ctypes.c_int),
    "pgcp_batch_stitch": ([_VP, _VP, ctypes.c_int, _D, _D, _VP, _VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "pgcp_batch_last_solve": ([_VP, ctypes.c_int, _PD, ctypes.c_int], ctypes.c_int),
    "pgcp_launch_count": ([], ctypes.c_ulonglong),
    "pgcp_workspace_stats": ([_PD, ctypes.c_int], ctypes.c_int),
    "pgcp_face_layout": ([_VP, _VP, _I64, _VP, _VP], ctypes.c_int),
    "pgcp_beltrami": ([_VP, _VP, _VP, _VP, _I64, _VP, _PI64, _VP], ctypes.c_int),
    "pgcp_corner_angles": ([_VP, ctypes.c_int, _VP, _I64, _VP, _VP, _VP], ctypes.c_int),
    "pgcp_area_distortion": ([_VP, _VP, _I64, _I64, _VP, ctypes.c_int, _VP, _VP, _VP], ctypes.c_int),
    "pgcp_batch_lbs_stiffness": ([_VP, _VP, _VP, _VP, _VP], ctypes.c_int),
    "pgcp_batch_qc_repair": ([_VP, _VP, _I32, _VP, _VP, _I64, _I32, _D, ctypes.POINTER(SolveOpts), _VP, _VP, _VP,
                              _VP], ctypes.c_int),
}

_OPTIONAL = {}


def lib():
    """Load (once) and return the native library; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1903_12359_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        for name, (args, res) in _OPTIONAL.items():
            if hasattr(L, name):
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
        if L.pgcp_abi_version() != 2:
            raise RuntimeError("libpgcp_b200.so ABI version mismatch")
        _lib = L
        return L


def register(name, args, res=ctypes.c_int):
    """Declare an additional entry point (used by modules added later)."""
    _OPTIONAL[name] = (args, res)
    if _lib is not None and hasattr(_lib, name):
        fn = getattr(_lib, name)
        fn.argtypes = args
        fn.restype = res


_EXC = {
    E_INVALID: ValueError,
    E_MESH: MeshError,
    E_PARTITION: PartitionError,
    E_SOLVE: SolveError,
    E_NOCONV: SolveError,
    E_WELD: WeldError,
    E_CUDA: RuntimeError,
    E_VALIDATION: ValidationError,
}


def check(status):
    if status == OK:
        return
    msg = lib().pgcp_last_error()
    msg = msg.decode(errors="replace") if msg else f"status {status}"
    raise _EXC.get(status, RuntimeError)(msg)

"""ctypes binding of libmsfv.so (include/msfv.h).

The product path has no CPU fallback: if the library is missing or CUDA is
unavailable, every entry point raises.  This module never touches the oracle.
"""

import ctypes
import os

from .errors import (FactorizationError, InvalidModelError, ReducedSingularError,
                     StaleBasisError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MSFV_LIB_PATH") or os.path.join(HERE, "libmsfv.so")   # override: A/B runs only

MSFV_OK = 0
MSFV_INVALID_MODEL = 1
MSFV_STALE_BASIS = 2
MSFV_REDUCED_SINGULAR = 3
MSFV_SHAPE = 4
MSFV_CUDA = 5
MSFV_FACTORIZATION = 6
MSFV_UNSUPPORTED = 7

FLAG_NONFINITE = 1
FLAG_NONPOSITIVE = 2
FLAG_LOCAL_NOT_SPD = 4
FLAG_COARSE_NOT_SPD = 8

INFO_NN, INFO_N, INFO_NCELLS, INFO_NEDGES, INFO_NBLOCKS, INFO_NI, INFO_P1S, INFO_K, \
    INFO_AK_DOUBLES, INFO_BASIS_SMEM, INFO_NT, INFO_PT, INFO_TB, INFO_PC, \
    INFO_FACTOR_DOUBLES, INFO_SCRATCH_DOUBLES, INFO_TC, INFO_COARSE, INFO_RED_FACE, INFO_RED_BOX = range(20)
INFO_COUNT = 20

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

# name -> (restype, argtypes)
SIGNATURES = {
    "msfv_abi_version": (ctypes.c_int, []),
    "msfv_last_error": (ctypes.c_char_p, []),
    "msfv_launch_count": (ctypes.c_int64, []),
    "msfv_plan_create": (ctypes.c_int, [_P, _P, _P, ctypes.POINTER(_P)]),
    "msfv_plan_destroy": (None, [_P]),
    "msfv_plan_info": (ctypes.c_int, [_P, _P, _I32]),
    "msfv_points_create": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, ctypes.POINTER(_P)]),
    "msfv_points_destroy": (None, [_P]),
    "msfv_operator": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "msfv_edge_average": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "msfv_basis_build": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    "msfv_basis_forward": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "msfv_basis_backward": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_basis_csc": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P]),
    "msfv_galerkin": (ctypes.c_int, [_P, _P, _D, _P, _P]),
    "msfv_coarse_diag": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_coarse_factor": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_coarse_solve": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv_survey_receive": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _P, _P]),
    "msfv_misfit": (ctypes.c_int, [_P, _P, ctypes.c_int64, _P, _P, _P]),
    "msfv_survey_restrict": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _P]),
    "msfv_survey_scatter": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "msfv_prolong": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "msfv_residual": (ctypes.c_int, [_P, _P, _D, _P, _P, _D, _I32, _P, _P]),
    "msfv_interior_solve": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv_restrict_op": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I32, _D, _P, _P, _P]),
    "msfv_cell_gradient": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I32, _P, _P, _P]),
    "msfv_points_interior_blocks": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "msfv_points_interior_scatter": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "msfv_points_interior_solve": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _P]),
    "msfv_block_gradient": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _P, _P]),
    "msfv_operator_slab": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _I32, _P]),
    "msfv_basis_forward_slab": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I32, _I32, _P]),
    "msfv_block_gradient_slab": (ctypes.c_int, [_P, _P, _P, _P, _P, _I32, _P, _P, _P, _P, _I32, _I32, _P, _P]),
    "msfv_jv_coarse_rhs": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _P, _P, _P, _P]),
    "msfv_coarse_dense": (ctypes.c_int, [_P, _P, _D, _P, _P]),
    "msfv_plan_set_reduced": (ctypes.c_int, [_P, _I32]),
    "msfv_boundary_reduced": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "msfv_plan_bind_boundary": (ctypes.c_int, [_P, _P]),
    "msfv_basis_csc_box": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P]),
    "msfv_plan_create_mesh": (ctypes.c_int, [_P, _P, ctypes.POINTER(_P)]),
    "msfv_fine_apply": (ctypes.c_int, [_P, _P, _P, _I32, _P, _P]),
    "msfv_full_gradient": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P, _P, _P]),
    "msfv_edge_grad": (ctypes.c_int, [_P, _P, _I32, _P, _P]),
    "msfv_edge_div": (ctypes.c_int, [_P, _P, _I32, _P, _P]),
    "msfv_cell_gather": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "msfv_reg_apply": (ctypes.c_int, [_P, _D, _P, _P, _P]),
    "msfv_reg_faces": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_yk_rhs": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "msfv_block_solve_compact": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv_yk_rowcount": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_yk_scatter": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "msfv_xk_present": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_xk_rowcount": (ctypes.c_int, [_P, _P, _P, _P]),
    "msfv_xk_values": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _P]),
    # 2D path (BASELINE configs 1-2)
    "msfv2d_plan_create": (ctypes.c_int, [_P, _P, _P, ctypes.POINTER(_P)]),
    "msfv2d_plan_destroy": (None, [_P]),
    "msfv2d_plan_info": (ctypes.c_int, [_P, _P, _I32]),
    "msfv2d_operator": (ctypes.c_int, [_P, _P, _P, _P, _P, _P]),
    "msfv2d_basis": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "msfv2d_galerkin": (ctypes.c_int, [_P, _P, _D, _P, _P]),
    "msfv2d_coarse_factor": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "msfv2d_coarse_solve": (ctypes.c_int, [_P, _P, _P, _I32, _P]),
    "msfv2d_interior_solve": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_prolong": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_restrict": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_apply_A": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_grad": (ctypes.c_int, [_P, _P, _P, _I32, _P]),
    "msfv2d_gradT": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_edge_average": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "msfv2d_cell_adjoint": (ctypes.c_int, [_P, _P, _P, _P, _I32, _P]),
    "msfv2d_spmm": (ctypes.c_int, [_I64, _P, _P, _P, _P, _I32, _D, _P, _P]),
    "msfv2d_axpby": (ctypes.c_int, [_I64, _D, _P, _P, _P, _P]),
    "msfv2d_fma3": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, _P, _P]),
}

_LIB = None


def load(path=LIB_PATH):
    """Load and type the shared library (no CUDA call is made here)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -m paper_1707_07598_b200.build` "
            "(the MSFV path has no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def last_error():
    msg = load().msfv_last_error()
    return msg.decode() if msg else ""


def check(rc, what=""):
    if rc == MSFV_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == MSFV_INVALID_MODEL:
        raise InvalidModelError(msg)
    if rc == MSFV_STALE_BASIS:
        raise StaleBasisError(msg)
    if rc == MSFV_REDUCED_SINGULAR:
        raise ReducedSingularError(msg)
    if rc == MSFV_SHAPE:
        raise ValueError(msg)
    if rc == MSFV_FACTORIZATION:
        raise FactorizationError(msg)
    if rc == MSFV_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)

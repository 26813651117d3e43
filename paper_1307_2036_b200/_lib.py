"""ctypes binding of libpmg.so (include/pmg.h).

There is no CPU fallback: importing the solver modules without the
built library, or calling a kernel without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMG_LIB", os.path.join(_HERE, "libpmg.so"))

PMG_OK = 0
PMG_ERR_VALUE = -1
PMG_ERR_CUDA = -2
PMG_ERR_PIVOT = -3
PMG_ERR_BREAKDOWN = -5
OFF = 4


class MGDesc(C.Structure):
    _fields_ = [
        ("nu_pre", C.c_int), ("nu_post", C.c_int), ("coarse_sweeps", C.c_int),
        ("rho", C.c_double), ("periodic_x", C.c_int), ("periodic_y", C.c_int),
        ("lagged_norm", C.c_int), ("red_restrict", C.c_int),
    ]


class PartDesc(C.Structure):
    _fields_ = [("worker", C.c_int), ("nbr", C.c_int * 4), ("diag", C.c_int * 4)]


class LevelDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("i0", C.c_int), ("j0", C.c_int),
        ("omega2", C.c_double), ("vcoef", C.c_double),
        ("dr", C.c_void_p), ("vprof", C.c_void_p), ("volprof", C.c_void_p),
        ("wx", C.c_void_p), ("wy", C.c_void_p), ("av", C.c_void_p),
        ("vh", C.c_void_p), ("sumw", C.c_void_p),
    ]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_LL = C.c_longlong

# name -> (restype, argtypes)
SIGNATURES = {
    "pmg_version": (_I, []),
    "pmg_launch_count": (_LL, []),
    "pmg_set_tracing": (_I, [_I]),
    "pmg_get_tracing": (_I, []),
    "pmg_last_error": (C.c_char_p, []),
    "pmg_device_sm_count": (_I, [_I, C.POINTER(_I)]),
    "pmg_level_create": (_I, [C.POINTER(LevelDesc), C.POINTER(_P)]),
    "pmg_level_destroy": (_I, [_P]),
    "pmg_level_field_doubles": (_LL, [_P]),
    "pmg_level_layout": (_I, [_P, C.POINTER(_I), C.POINTER(_LL), C.POINTER(_LL),
                              C.POINTER(_I), C.POINTER(_I)]),
    "pmg_level_tables": (_I, [_P, _P, _P, _P]),
    "pmg_level_prepare": (_I, [_P, _P]),
    "pmg_level_dims": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "pmg_field_upload": (_I, [_P, _P, _P, _P, _P]),
    "pmg_field_download": (_I, [_P, _P, _P, _P, _P]),
    "pmg_fill": (_I, [_P, _P, _D, _P]),
    "pmg_copy": (_I, [_P, _P, _P, _P]),
    "pmg_copy_block": (_I, [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "pmg_norm2": (_I, [_P, _P, _P, _P, _P]),
    "pmg_ssor_apply": (_I, [_P, _P, _P, _D, _I, _I, _P, _P, _P]),
    "pmg_hier_create": (_I, [C.POINTER(_P), _I, C.POINTER(MGDesc), C.POINTER(_P)]),
    "pmg_hier_destroy": (_I, [_P]),
    "pmg_hier_graph_launches": (_LL, [_P, _P, _P, _I]),
    "pmg_hier_replayed_launches": (_LL, [_P]),
    "pmg_hier_cycle_times": (_I, [_P, _P, _I]),
    "pmg_vcycle": (_I, [_P, _P, _P, _I, _P]),
    "pmg_mg_solve": (_I, [_P, _P, _P, _D, _I, _P, C.POINTER(_I), C.POINTER(_I), _P]),
    "pmg_pcg_work_doubles": (_LL, [_P]),
    "pmg_pcg_solve": (_I, [_P, _P, _P, _D, _I, _D, _I, _D, _I, _I, _P, _P, C.POINTER(_I),
                           C.POINTER(_I), _P]),
    "pmg_from_ref_layout": (_I, [_P, _P, _P, _P]),
    "pmg_to_ref_layout": (_I, [_P, _P, _P, _P]),
    "pmg_from_ref_layout_slab": (_I, [_P, _P, _P, C.c_int, C.c_int, _P]),
    "pmg_to_ref_layout_slab": (_I, [_P, _P, _P, C.c_int, C.c_int, _P]),
    "pmg_apply": (_I, [_P, _P, _P, _P]),
    "pmg_residual": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "pmg_apply_dot": (_I, [_P, _P, _P, _P, _P, _P]),
    "pmg_residual_restrict": (_I, [_P, _P, _P, _P, _P, _P]),
    "pmg_residual_restrict_red": (_I, [_P, _P, _P, _P, _P, _P]),
    "pmg_residual_restrict_red_ok": (_I, [_P]),
    "pmg_red_residual_norm": (_I, [_P, _P, _P, _P, _P, _P]),
    "pmg_half_sweep": (_I, [_P, _P, _P, _I, _D, _I, _I, _D, _P]),
    "pmg_half_sweep_res": (_I, [_P, _P, _P, _P, _P, _P, _P]),
    "pmg_half_sweep_region_ok": (_I, [_P]),
    "pmg_half_sweep_region": (_I, [_P, _P, _P, _I, _D, _I, _I, _D, _I, _I, _I, _I, _I, _I, _P]),
    "pmg_half_sweep_res_ok": (_I, [_P]),
    "pmg_set_smoother_mode": (_I, [_I]),
    "pmg_get_smoother_mode": (_I, []),
    "pmg_restrict": (_I, [_P, _P, _P, _P, _D, _P]),
    "pmg_prolong": (_I, [_P, _P, _P, _P, _I, _P]),
    "pmg_prolong_add": (_I, [_P, _P, _P, _P, _P]),
    "pmg_field_alloc": (_I, [_P, _P]),
    "pmg_field_free": (_I, [_P]),
    "pmg_prolong_colors": (_I, [_P, _P, _P, _P, _I, _I, _P]),
    "pmg_halo_self": (_I, [_P, _P, _I, _I, _P]),
    "pmg_face_doubles": (_LL, [_P, _I]),
    "pmg_pack_face": (_I, [_P, _P, _I, _P, _P]),
    "pmg_unpack_face": (_I, [_P, _P, _I, _P, _I, _P]),
    "pmg_partials_size": (_LL, []),
    "pmg_dot": (_I, [_P, _P, _P, _P, _P, _P]),
    "pmg_axpy": (_I, [_LL, _D, _P, _P, _P]),
    "pmg_xpby": (_I, [_LL, _P, _D, _P, _P]),
    "pmg_cg_update": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pmg_cg_direction": (_I, [_LL, _P, _P, _P, _P, _P]),
    "pmg_cg_step": (_I, [_LL, _P, _P, _P, _P, _P, _P, _P, _P]),
    "pmg_thomas_batch": (_I, [_I, _LL, _P, _P, _P, _P, _P, _P, C.POINTER(_I), _P]),
    "pmg_thomas_work_doubles": (_LL, [_I, _LL]),
    "pmg_comm_available": (_I, []),
    "pmg_comm_unique_id": (_I, [_P]),
    "pmg_comm_create": (_I, [_P, _I, _I, C.POINTER(_P)]),
    "pmg_comm_destroy": (_I, [_P]),
    "pmg_exchange_plan": (_I, [C.POINTER(_I), _I, C.POINTER(_I), C.POINTER(_I)]),
    "pmg_exchange_plan8": (_I, [C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "pmg_phier_create": (_I, [C.POINTER(_P), _I, _I, C.POINTER(PartDesc), C.POINTER(MGDesc), _P,
                              _I, C.POINTER(_P)]),
    "pmg_phier_destroy": (_I, [_P]),
    "pmg_phier_mg_solve": (_I, [_P, C.POINTER(_P), C.POINTER(_P), _D, _I, _P, C.POINTER(_I),
                                C.POINTER(_I), _P]),
    "pmg_phier_vcycle": (_I, [_P, C.POINTER(_P), C.POINTER(_P), _I, _P]),
    "pmg_phier_pcg_solve": (_I, [_P, C.POINTER(_P), C.POINTER(_P), _D, _I, _D, _I, _D, _P,
                                 C.POINTER(_I), C.POINTER(_I), _P]),
    "pmg_phier_halo_exchange": (_I, [_P, _I, C.POINTER(_P), _P]),
    "pmg_phier_dot": (_I, [_P, _I, C.POINTER(_P), C.POINTER(_P), _P, _P]),
    "pmg_phier_replayed_launches": (_LL, [_P]),
    "pmg_phier_cycle_times": (_I, [_P, _P, _I]),
    "pmg_phier_exchanges": (_LL, [_P]),
}


class PivotError(ArithmeticError):
    pass


_lib = None


def load():
    """Load libpmg.so (built by ``__graft_entry__.build()``); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libpmg.so not found at {LIB_PATH}: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = ""):
    if rc == PMG_OK:
        return
    msg = load().pmg_last_error().decode(errors="replace")
    if rc == PMG_ERR_VALUE:
        raise ValueError(f"{what}: {msg}")
    if rc == PMG_ERR_PIVOT:
        from .tridiag import ZeroPivotError
        raise ZeroPivotError(f"{what}: {msg}")
    if rc == PMG_ERR_BREAKDOWN:
        from .krylov import BreakdownError
        raise BreakdownError(msg)
    raise RuntimeError(f"{what}: {msg}")


def call(name: str, *args):
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc


# Library objects whose destruction was requested while the current stream
# was being captured (a garbage-collected hierarchy or level inside a
# ``torch.cuda.graph`` block): their cudaFree would invalidate the capture,
# so they wait here until a destructor runs outside one.
_PENDING: list = []


def _capturing() -> bool:
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.is_current_stream_capturing()
    except Exception:                                   # interpreter shutdown
        return False


def destroy(name: str, handle) -> None:
    """Call the destructor ``name`` on ``handle`` -- now, or once no stream
    capture is under way."""
    if _lib is None:
        return
    if _capturing():
        _PENDING.append((name, handle))
        return
    while _PENDING:
        n, h = _PENDING.pop()
        getattr(_lib, n)(h)
    getattr(_lib, name)(handle)

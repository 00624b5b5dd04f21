"""ctypes binding of libhevi.so (the C ABI declared in include/hevi.h).

There is no fallback: if the library is missing or no CUDA device is
present, every compute entry point raises.  ``load()`` only needs the .so
(CPU hosts can load it to check the exported symbols).
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEVI_LIB") or os.path.join(_HERE, "_lib", "libhevi.so")

HEVI_OK = 0
F_NONFINITE_OUT = 1 << 12
F_PIVOT = 1 << 13
F_AINV = 1 << 14
STEP_PP_VALID = 1
STAGE_INTERIOR = 2
STAGE_BOUNDARY = 4


def F_NONFINITE_IN(stage):
    return 1 << (stage * 4 + 0)


def F_EOS(stage):
    return 1 << (stage * 4 + 1)


class GridDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in (
        "nex", "ney", "nez", "N", "Ny", "slab", "x0", "y0", "lX", "lY", "px",
        "ex_b", "ex_e", "ey_b", "ey_e")]


_DP = ctypes.POINTER(ctypes.c_double)


class RefDesc(ctypes.Structure):
    _fields_ = [(n, _DP) for n in (
        "rho0", "theta0", "P0f", "drho0", "dtheta0", "G0", "H0", "F0z", "rho0G0", "Pb",
        "cx", "cy", "cz", "Dx", "Dy", "Dz", "Theta0", "F0c")] + [
        (n, ctypes.c_double) for n in ("g", "R", "P0", "gamma")] + [("eqset", ctypes.c_int)]


_IP = ctypes.POINTER(ctypes.c_int)


class GMeshDesc(ctypes.Structure):
    """hevi_gmesh_desc: general (curvilinear) mesh, host arrays."""
    _fields_ = [("nel", ctypes.c_int), ("N", ctypes.c_int)] + [
        (n, _DP) for n in ("D", "ar", "as_", "at", "vert", "Jtv", "w")] + [
        ("n_groups", ctypes.c_int), ("grp_ptr", _IP), ("grp_idx", _IP), ("grp_wsum", _DP),
        ("n_proj", ctypes.c_int), ("grp_slot", _IP), ("proj", _DP),
        ("n_col", ctypes.c_int), ("n_lev", ctypes.c_int), ("uid", _IP), ("rep", _IP)]


class GRefDesc(ctypes.Structure):
    """hevi_gref_desc: per-node background."""
    _fields_ = [(n, _DP) for n in (
        "rho0", "theta0", "P0f", "grad_rho0", "grad_theta0", "gvec", "G0", "H0", "F0vec",
        "Theta0", "F0c", "Pb")] + [
        (n, ctypes.c_double) for n in ("g", "R", "P0", "gamma")] + [("eqset", ctypes.c_int)]


# exported symbol -> (restype, argtypes); this list IS the C ABI of hevi.h
_V = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_LL = ctypes.c_longlong
SIGNATURES = {
    "hevi_plan_create": (_I, [ctypes.POINTER(_V), ctypes.POINTER(GridDesc), ctypes.POINTER(RefDesc)]),
    "hevi_plan_destroy": (_I, [_V]),
    "hevi_last_error": (ctypes.c_char_p, []),
    "hevi_state_size": (_LL, [_V]),
    "hevi_factor": (_I, [_V, _D, ctypes.POINTER(_I), _V]),
    "hevi_column_matrix": (_I, [_V, _D, _V, _V, _V]),
    "hevi_rhs": (_I, [_V, _V, _V, _V]),
    "hevi_linear_v": (_I, [_V, _V, _V, _V]),
    "hevi_solve": (_I, [_V, _D, _V, _V, _V]),
    "hevi_stage": (_I, [_V, _I, _D, _V, _V, _V, _V]),
    "hevi_stage_solve": (_I, [_V, _I, _D, _V, _V]),
    "hevi_ark2_step": (_I, [_V, _D, _V, _V, _V, _V]),
    "hevi_ark2_step_ex": (_I, [_V, _D, _V, _V, _V, ctypes.c_uint, _V]),
    "hevi_pp_refresh": (_I, [_V, _V, _V, _V]),
    "hevi_stage_ex": (_I, [_V, _I, _D, _V, _V, _V, ctypes.c_uint, _V]),
    "hevi_step_chains_pp": (_I, [_V]),
    "hevi_stage_tiles": (_I, [_V, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "hevi_rk35_step": (_I, [_V, _D, _V, _V, _V]),
    "hevi_evec_to_lattice": (_I, [_V, _V, _V, _I, _V]),
    "hevi_lattice_to_evec": (_I, [_V, _V, _V, _I, _V]),
    "hevi_flags": (_I, [_V, ctypes.POINTER(ctypes.c_uint), _I, _V]),
    "hevi_band_pack": (_I, [_V, _V, _I, _I, _I, _V]),
    "hevi_band_unpack": (_I, [_V, _V, _I, _I, _I, _V]),
    "hevi_band_lu": (_I, [_V, _I, _I, _I, _D, ctypes.POINTER(_I), _V]),
    "hevi_band_solve": (_I, [_V, _V, _I, _I, _I, _V]),
    "hevi_absmax": (_I, [_V, _LL, ctypes.POINTER(_D), _V]),
    "hevi_lu_pivot": (_I, [_V, _V, _I, _I, _V, _V]),
    "hevi_diagnostics": (_I, [_V, _V, _V, _V, _V, _V, _V]),
    "hevi_std_solve": (_I, [_V, _V, _I, _I, _V, _V, _V]),
    "hevi_halo_pack": (_I, [_V, _V, _I, _I, _I, _I, _I, _V, _V]),
    "hevi_halo_unpack": (_I, [_V, _V, _I, _I, _I, _I, _I, _V, _V]),
    "hevi_linear3": (_I, [_V, _V, _V, _V]),
    "hevi_grad": (_I, [_V, _I, _V, _V, _V]),
    "hevi_div": (_I, [_V, _I, _V, _V, _V]),
    "hevi_dss": (_I, [_V, _V, _V, _I, _V, _V, _V, _V]),
    "hevi_schur3_up": (_I, [_V, _D, _I, _V, _V, _V]),
    "hevi_schur3_flux": (_I, [_V, _D, _I, _V, _V, _V, _V]),
    "hevi_schur3_ua": (_I, [_V, _D, _V, _V, _V, _V]),
    "hevi_schur3_extract": (_I, [_V, _D, _V, _V, _V, _V, _V, _V]),
    "hevi_wdot": (_I, [_V, _V, _V, _I, _V, _V]),
    "hevi_axpby": (_I, [_LL, _D, _V, _D, _V, _V]),
    "hevi_lu_pivot_solve": (_I, [_V, _V, _V, _I, _I, _V]),
    "hevi_plan_set_option": (_I, [_V, _I, _I]),
    "hevi_factor_pivoted": (_I, [_V, _D, ctypes.POINTER(_I)]),
    # general (curvilinear) meshes: the cubed-sphere shell
    "hevi_gplan_create": (_I, [ctypes.POINTER(_V), ctypes.POINTER(GMeshDesc), ctypes.POINTER(GRefDesc)]),
    "hevi_gplan_destroy": (_I, [_V]),
    "hevi_g_work_fields": (_I, [_V]),
    "hevi_g_rhs": (_I, [_V, _V, _V, _V]),
    "hevi_g_linear_v": (_I, [_V, _V, _V, _V]),
    "hevi_g_factor": (_I, [_V, _D, ctypes.POINTER(_I), ctypes.POINTER(_I), _V]),
    "hevi_g_column_matrix": (_I, [_V, _D, _I, _V, _V]),
    "hevi_g_solve": (_I, [_V, _D, _V, _V, _V]),
    "hevi_g_ark2_step": (_I, [_V, _D, _V, _V, _V, _V]),
    "hevi_g_rk35_step": (_I, [_V, _D, _V, _V, _V]),
    "hevi_g_dss": (_I, [_V, _V, _V, _I, _V]),
    "hevi_g_grad": (_I, [_V, _I, _V, _V, _V]),
    "hevi_g_div": (_I, [_V, _I, _V, _V, _V]),
    "hevi_g_flags": (_I, [_V, ctypes.POINTER(ctypes.c_uint), _I, _V]),
    "hevi_g_schur3_ua": (_I, [_V, _D, _V, _V, _V, _V]),
    "hevi_g_schur3_up": (_I, [_V, _D, _I, _V, _V, _V]),
    "hevi_g_schur3_flux": (_I, [_V, _D, _I, _V, _V, _V, _V]),
    "hevi_g_schur3_extract": (_I, [_V, _D, _I, _V, _V, _V, _V, _V, _V]),
    "hevi_g_linear3": (_I, [_V, _V, _V, _V]),
    "hevi_g_dot": (_I, [_V, _V, _V, _LL, ctypes.POINTER(_D), _V]),
}

_lib = None


class NativeMissing(RuntimeError):
    pass


def load():
    """Load libhevi.so (raises NativeMissing if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeMissing(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc):
    if rc != HEVI_OK:
        msg = load().hevi_last_error().decode()
        raise RuntimeError(f"libhevi error {rc}: {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("the HEVI path runs on a CUDA device only (no CPU fallback); "
                           "torch.cuda.is_available() is False")
    load()


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    """Device pointer of a contiguous float64 CUDA tensor."""
    return ctypes.c_void_p(t.data_ptr())

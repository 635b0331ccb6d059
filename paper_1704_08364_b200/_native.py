"""ctypes binding of the sm_100a library behind ``include/tb_bst.h``.

This is the ONLY way the package computes: there is no CPU or PyTorch
fallback.  If ``lib/libtb_bst.so`` is missing the import of the compute
entry points raises immediately (build it with ``make`` or
``python -c "import __graft_entry__ as g; g.build()"``).
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIB_PATH") or os.path.join(HERE, "lib", "libtb_bst.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "tb_bst.h")

TB_OK = 0
TB_ERR_INVALID = 1
TB_ERR_UNSUPPORTED = 2
TB_ERR_CUDA = 3
TB_ERR_WORKSPACE = 4
TB_ERR_NONFINITE_INPUT = 5
TB_ERR_NONFINITE_OUTPUT = 6


class tb_plan_desc(ctypes.Structure):
    _fields_ = [
        ("n_t", ctypes.c_int32),
        ("n_theta", ctypes.c_int32),
        ("pad_factor", ctypes.c_int32),
        ("radial_samples", ctypes.c_int32),
        ("kb_beta", ctypes.c_double),
        ("kb_support", ctypes.c_double),
        ("sigma_min_bins", ctypes.c_int32),
        ("interp", ctypes.c_int32),
        ("output_n", ctypes.c_int32),
        ("full_turn", ctypes.c_int32),
        ("filter_kind", ctypes.c_int32),
        ("rolloff", ctypes.c_double),
        ("n_angles", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


TB_PLAN_NO_GRID = 1


class tb_plan_info(ctypes.Structure):
    _fields_ = [
        ("n_t", ctypes.c_int32),
        ("n_theta", ctypes.c_int32),
        ("n_angles", ctypes.c_int32),
        ("radial_samples", ctypes.c_int32),
        ("ramp_samples", ctypes.c_int32),
        ("output_n", ctypes.c_int32),
        ("support_lo", ctypes.c_int32),
        ("support_hi", ctypes.c_int32),
        ("amplitude_scale", ctypes.c_double),
    ]


class tb_workspace_layout(ctypes.Structure):
    _fields_ = [(k, ctypes.c_size_t) for k in
                ("total", "polar", "rowcoef", "common", "coefmean", "columns", "filtered", "status")]


_lib = None
_lock = threading.Lock()


class NativeLibraryMissing(RuntimeError):
    pass


def _bind(lib):
    P = ctypes.c_void_p
    I = ctypes.c_int
    S = ctypes.c_size_t
    sig = {
        "tb_abi_version": (I, []),
        "tb_last_error": (ctypes.c_char_p, []),
        "tb_plan_create": (I, [ctypes.POINTER(tb_plan_desc), I, ctypes.POINTER(P)]),
        "tb_plan_destroy": (I, [P]),
        "tb_plan_get_info": (I, [P, ctypes.POINTER(tb_plan_info)]),
        "tb_workspace_bytes": (I, [P, I, ctypes.POINTER(S)]),
        "tb_workspace_get_layout": (I, [P, I, ctypes.POINTER(tb_workspace_layout)]),
        "tb_fbp": (I, [P, P, P, I, I, P, S, P]),
        "tb_bst": (I, [P, P, P, I, I, P, S, P]),
        "tb_bst_scaled": (I, [P, P, P, I, I, P, S, ctypes.c_float, P]),
        "tb_fbp_profiled": (I, [P, P, P, I, I, P, S, P, ctypes.POINTER(ctypes.c_double)]),
        "tb_ramp": (I, [P, P, P, I, P]),
        "tb_ss": (I, [P, P, P, I, ctypes.c_float, P]),
        "tb_fbp_ss": (I, [P, P, P, I, I, P, S, P]),
        "tb_fbp_counts": (I, [P, P, P, P, ctypes.c_double, P, I, I, P, S, P]),
        "tb_fbp_frames": (I, [P, P, P, I, I, P, S, P]),
        "tb_fbp_counts_const": (I, [P, P, ctypes.c_double, ctypes.c_double, ctypes.c_double, P, I, I, P, S, P]),
        "tb_normalize": (I, [P, P, P, P, ctypes.c_double, P, I, P]),
        "tb_forward": (I, [P, P, P, I, ctypes.c_double, I, P]),
        "tb_center_estimate": (I, [P, P, I, P, P, P]),
        "tb_center_apply": (I, [P, P, P, P, I, P]),
        "tb_rings": (I, [P, P, P, I, P, I, P]),
        "tb_pre_params": (I, [P, P, I, P, I, P, P, P, P]),
        "tb_fbp_pre": (I, [P, P, P, I, I, P, S, P, P, P]),
        "tb_copy_polar": (I, [P, P, I, P, P]),
        "tb_reset_status": (I, [P, P, P]),
        "tb_read_status": (I, [P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


def lib():
    """The loaded native library (raises NativeLibraryMissing if absent)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeLibraryMissing(
                        f"native library {LIB_PATH} is missing: build it with `make` "
                        "(there is no CPU fallback)")
                _lib = _bind(ctypes.CDLL(LIB_PATH))
    return _lib


def header_functions() -> list[str]:
    """Names of every function declared in include/tb_bst.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(tb_\w+)\s*\(", text, re.M)))


def last_error() -> str:
    return lib().tb_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a tb_status to the reference's exception types
    (ValueError / FloatingPointError, fourier_bp.py:89-109, 459-460)."""
    if rc == TB_OK:
        return
    msg = last_error()
    if rc == TB_ERR_INVALID:
        raise ValueError(msg)
    if rc == TB_ERR_NONFINITE_INPUT:
        raise ValueError(msg)
    if rc == TB_ERR_NONFINITE_OUTPUT:
        raise FloatingPointError(msg)
    if rc == TB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"{what}: {msg} (status {rc})")

"""ctypes binding of libbnff.so (include/bnff.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a) and
loaded from this package directory.  There is no fallback: if the library is
missing or the device is not sm_100, ``lib()`` raises -- the product path never
silently drops to a CPU or PyTorch implementation.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import EngineError, ShapeError, StateError, UnsupportedError

_HERE = os.path.dirname(os.path.abspath(__file__))
# BNFF_LIB selects another build of the same ABI (A/B timing of kernel variants on one box)
LIB_PATH = os.environ.get("BNFF_LIB") or os.path.join(_HERE, "libbnff.so")

F32, BF16 = 0, 1
PRO_NONE, PRO_RELU, PRO_BN_RELU, PRO_BN_DX = 0, 1, 2, 3
DG_PLAIN, DG_CLIP, DG_NRC, DG_NRC_ACC, DG_NRC_SET = 0, 1, 2, 3, 4
WT_FPROP_PRO, WT_DGRAD_NRC, WT_DGRAD_PRO = 1, 2, 4  # bnff_window_ok_ex table flags
WT_ALL = WT_FPROP_PRO | WT_DGRAD_NRC | WT_DGRAD_PRO


class View(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("n", C.c_int64), ("h", C.c_int64), ("w", C.c_int64),
                ("c", C.c_int64), ("row_stride", C.c_int64)]


class Coef(C.Structure):
    _fields_ = [("a", C.c_void_p), ("b", C.c_void_p), ("c", C.c_void_p), ("d", C.c_void_p),
                ("e", C.c_void_p)]


class FpropArgs(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32),
                ("pad", C.c_int32), ("x", View), ("y", View), ("wpack", C.c_void_p),
                ("bias", C.c_void_p), ("x_pro", C.c_int32), ("x_coef", Coef),
                ("stat_part", C.c_void_p), ("wwin", C.c_void_p)]


class DgradArgs(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32),
                ("pad", C.c_int32), ("dy", View), ("dy_x", View), ("dy_pro", C.c_int32),
                ("dy_coef", Coef), ("dx", View), ("x", View), ("wpack_t", C.c_void_p),
                ("epi", C.c_int32), ("x_coef", Coef), ("stat_part", C.c_void_p),
                ("wwin", C.c_void_p)]


class WgradArgs(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32),
                ("pad", C.c_int32), ("x", View), ("x_pro", C.c_int32), ("x_coef", Coef),
                ("dy", View), ("dy_x", View), ("dy_pro", C.c_int32), ("dy_coef", Coef),
                ("splits", C.c_int32), ("workspace", C.c_void_p), ("dw", C.c_void_p),
                ("dw_cin", C.c_int32), ("dbias", C.c_void_p)]


class PackJob(C.Structure):
    _fields_ = [("w", C.c_void_p), ("wfwd", C.c_void_p), ("wdgrad", C.c_void_p),
                ("c_out", C.c_int32), ("c_in", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32)]


class GradTerm(C.Structure):
    _fields_ = [("g", View), ("x", View), ("deferred", C.c_int32), ("coef", Coef)]


# exported symbols and their signatures (every name declared in include/bnff.h)
_I32, _I64, _P, _F, _D = C.c_int32, C.c_int64, C.c_void_p, C.c_float, C.c_double
SIGNATURES = {
    "bnff_last_error": (C.c_char_p, []),
    "bnff_version": (C.c_int, []),
    "bnff_device_ok": (C.c_int, []),
    "bnff_stat_rows": (_I32, []),
    "bnff_conv_fprop": (C.c_int, [C.POINTER(FpropArgs), _P]),
    "bnff_conv_dgrad": (C.c_int, [C.POINTER(DgradArgs), _P]),
    "bnff_wgrad_workspace": (_I64, [_I32] * 8),
    "bnff_conv_wgrad": (C.c_int, [C.POINTER(WgradArgs), _P]),
    "bnff_wgrad_default_splits": (_I32, [_I32] * 7),
    "bnff_pack_size": (_I64, [_I32] * 5),
    "bnff_pack_weights": (C.c_int, [_I32, _P, _I32, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "bnff_window_ok": (C.c_int, [_I32] * 9),
    "bnff_window_ok_ex": (C.c_int, [_I32] * 10),
    "bnff_window_pack_size": (_I64, [_I32] * 6),
    "bnff_pack_window": (C.c_int, [_I32, _P, _I32, _I32, _I32, _I32, _P, _P, _P]),
    "bnff_window_conv": (C.c_int, [_I32, _I32, _I32, _I32, View, View, _I32, Coef, View, _P, _P, _I32,
                                   View, Coef, _P, _P]),
    "bnff_window_wgrad_ws": (_I64, [_I32] * 6),
    "bnff_pack_window_multi": (C.c_int, [_I32, _I32, _P, _I64, _P]),
    "bnff_window_wgrad": (C.c_int, [View, _I32, Coef, View, View, _I32, Coef, _I32, _P, _P, _I32,
                                    _P, _P]),
    "bnff_sum_tiles": (_I32, [_I64]),
    "bnff_channel_sums": (C.c_int, [_I32, _I32, View, View, Coef, _P, _P]),
    "bnff_stats_finalize": (C.c_int, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _P]),
    "bnff_centered_var": (C.c_int, [_I32, View, _P, _P, _P]),
    "bnff_var_finalize": (C.c_int, [_P, _I32, _I32, _I64, _P, _P]),
    "bnff_var_finalize_coeffs": (C.c_int, [_P, _I32, _I32, _I64, _P, _P, _P, _P, C.c_float, _P, _P, _P, _P, _P]),
    "bnff_stats_finalize_coeffs": (C.c_int, [_P, _I32, _I32, _I64, _P, _P, _P, _P, _I32, _I32, _P, _P, _P,
                                             _P, _F, _P, _P, _P, _P, _P]),
    "bnff_bn_coeffs": (C.c_int, [_I32, _P, _P, _P, _P, _F, _P, _P, _P, _P, _P]),
    "bnff_dx_coeffs": (C.c_int, [_I32, _P, _I32, _I64, _P, _P, _P, _F, _P, _P, _P, _P, _P, _P,
                                 _P, _P, _P, _P]),
    "bnff_dx_coeffs_acc": (C.c_int, [_I32, _P, _I32, _I64, _P, _P, _P, _F, _P, _P, _P, _P, _P, _P,
                                     _P, _P, _P, _P, _P, _I32, _P]),
    "bnff_stats_from_sums": (C.c_int, [_I32, _I64, _P, _P, _P, _P, _P]),
    "bnff_dx_coeffs_from_sums": (C.c_int, [_I32, _I64, _P, _P, _P, _P, _P, _F, _P, _P, _P, _P, _P,
                                           _P]),
    "bnff_sums_to_f32": (C.c_int, [_I32, _P, _P, _P, _P, _P]),
    "bnff_bn_apply": (C.c_int, [_I32, View, View, Coef, _I32, _P]),
    "bnff_grad_sum": (C.c_int, [_I32, View, _I32, C.POINTER(GradTerm), _I32, _P]),
    "bnff_relu_fwd": (C.c_int, [_I32, View, View, _P]),
    "bnff_relu_bwd": (C.c_int, [_I32, View, View, View, _P]),
    "bnff_avgpool_fwd": (C.c_int, [_I32, View, View, _I32, _P, _P]),
    "bnff_norm_relu_pool_fwd": (C.c_int, [_I32, View, View, _I32, Coef, _P, _P]),
    "bnff_pool_relu_bn_bwd": (C.c_int, [_I32, View, View, View, _I32, Coef, _P, _P]),
    "bnff_avgpool_bwd": (C.c_int, [_I32, View, View, _I32, _P]),
    "bnff_ews_fwd": (C.c_int, [_I32, View, View, View, _P]),
    "bnff_copy": (C.c_int, [_I32, View, View, _P]),
    "bnff_nchw_to_nhwc": (C.c_int, [_I32, _P, _I64, _I64, _I64, _I64, View, _P]),
    "bnff_nhwc_to_nchw": (C.c_int, [_I32, View, _P, _P]),
    "bnff_sgd": (C.c_int, [_P, _P, _I64, _F, _P]),
    "bnff_debug_trace": (C.c_int, [_P]),
    "bnff_debug_mark": (C.c_int, [_I32, _P]),
    "bnff_im2col": (C.c_int, [_I32, View, _I32, _I32, _I32, _I32, _I32, View, _P]),
    "bnff_col2im": (C.c_int, [_I32, View, _I32, _I32, _I32, _I32, _I32, View, _P]),
    "bnff_im2col_s": (C.c_int, [_I32, View, _I32, _I32, _I32, _I32, _I32, Coef, View, _P]),
    "bnff_col2im_s": (C.c_int, [_I32, View, _I32, _I32, _I32, _I32, _I32, View, Coef, View, _P]),
    "bnff_weight_to_cols": (C.c_int, [_P, _I32, _I32, _I32, _I32, _I32, _P, _P]),
    "bnff_cols_to_weight": (C.c_int, [_P, _I32, _I32, _I32, _I32, _I32, _P, _P]),
}

_LIB = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """dlopen libbnff and attach signatures (no device call)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise EngineError(f"libbnff.so not built at {path}; run __graft_entry__.build()")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def lib() -> C.CDLL:
    """The loaded library, after checking the current device is an sm_100 part."""
    L = load()
    if not getattr(lib, "_checked", False):
        import torch
        if not torch.cuda.is_available():
            raise EngineError("libbnff needs a CUDA device (sm_100a); none is visible")
        torch.cuda.init()
        if L.bnff_device_ok() != 1:
            cap = torch.cuda.get_device_capability()
            raise EngineError(f"libbnff is built for sm_100a; device capability is {cap}")
        lib._checked = True
    return L


_ERRS = {1: ShapeError, 2: StateError, 3: UnsupportedError}


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = load().bnff_last_error().decode(errors="replace")
        raise _ERRS.get(rc, EngineError)(f"{what}: {msg}" if what else msg)
    return rc

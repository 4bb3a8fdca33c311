"""ctypes loader for libmasq.so (the C ABI declared in include/masq.h).

The product path has no fallback: if the shared library is missing or does not load,
every call raises.  Build it with `python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmasq.so")

c_void_p = ctypes.c_void_p
c_int32 = ctypes.c_int32
c_int64 = ctypes.c_int64
c_size_t = ctypes.c_size_t

# name -> (restype, argtypes) — mirrors include/masq.h exactly
SIGNATURES = {
    "masq_workspace_size": (c_size_t, [c_int32, c_int64, c_int64, c_int64, c_int32, c_int32]),
    "masq_calibrate_stats": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32,
                                       c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "masq_init_factors": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_int64, c_int32,
                                    c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_quantize_weight": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int64, c_int32,
                                       c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_quantize_activations": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32,
                                            c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                            c_size_t, c_void_p]),
    "masq_linear_forward": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                      c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                      c_void_p, c_void_p, c_int64, c_int32,
                                      c_void_p, c_int64, c_void_p, c_size_t, c_void_p, c_void_p]),
    "masq_reference_output": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64,
                                        c_void_p, c_int64, c_void_p, c_size_t, c_void_p]),
    "masq_calib_loss": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                  c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p,
                                  c_void_p, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_void_p, c_size_t, c_void_p]),
    "masq_loss_finalize": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p, c_void_p]),
    "masq_calib_loss_grad": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                       c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p,
                                       c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_cmc_factors": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                   c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_int32, ctypes.c_double,
                                   c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_quantize_weight_int4": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                                            c_void_p, c_void_p]),
    "masq_unpack_int4": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p]),
    "masq_linear_decode": (c_int32, [c_void_p, c_int32, c_int64, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                                     c_void_p, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_size_t, c_void_p]),
    "masq_quantize_weight_w4g": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                                           c_void_p, c_void_p]),
    "masq_linear_forward_w4g": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32,
                                          c_void_p, c_void_p, c_void_p, c_int32, c_int32,
                                          c_void_p, c_void_p, c_int64, c_int32,
                                          c_void_p, c_int64, c_void_p, c_size_t, c_void_p, c_void_p]),
    "masq_cmc_gram": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p,
                                c_int32, c_void_p, c_size_t, c_void_p]),
    "masq_cmc_factors_from_gram": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p, c_int32,
                                             c_void_p, c_void_p, c_int32, ctypes.c_double, c_void_p, c_void_p,
                                             c_int32, c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_smooth_factors": (c_int32, [c_void_p, c_int64, c_int64, c_void_p, ctypes.c_double, c_void_p, c_void_p]),
    "masq_calibrate_meanabs": (c_int32, [c_void_p, c_int32, c_int64, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_size_t, c_void_p]),
    "masq_count_modalities": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_int32, c_void_p, c_size_t,
                                        c_void_p]),
    "masq_range_stats": (c_int32, [c_void_p, c_int32, c_int64, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                                   c_void_p]),
    "masq_calib_layer": (c_int32, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_int32, c_void_p,
                                   c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int64, c_int32, c_void_p,
                                   c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_size_t, c_void_p]),
    "masq_adam_init": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "masq_keep_best": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "masq_adam_step": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double, c_void_p, c_void_p]),
    "masq_check": (c_int32, [c_void_p, c_void_p]),
    "masq_profile_enable": (c_int32, [c_int32]),
    "masq_profile_only": (c_int32, [ctypes.c_char_p]),
    "masq_profile_collect": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p]),
    "masq_status_string": (ctypes.c_char_p, [c_int32]),
    "masq_version": (ctypes.c_char_p, []),
}


class MasqDebug(ctypes.Structure):
    _fields_ = [("acc", c_void_p), ("ld_acc", c_int64), ("qx", c_void_p), ("dx", c_void_p)]


_lib = None


def lib():
    """Load libmasq.so once; raise loudly when it is missing (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libmasq.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib

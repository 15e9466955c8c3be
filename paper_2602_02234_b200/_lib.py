"""ctypes binding of libhmdp.so (the C-ABI in include/hmdp.h).

The library is built in-tree by build.py.  Loading it does not need a GPU (so
the CPU test suite can check the exported symbols and the host fixtures), but
every compute entry point needs a CUDA device and fails loudly without one:
there is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libhmdp.so")

HMDP_OK = 0
HMDP_INVALID_ARGUMENT = 1
HMDP_RUNTIME_ERROR = 2
HMDP_CUDA_ERROR = 3
HMDP_FP32 = 0
HMDP_FP64 = 1


class HmdpCudaError(RuntimeError):
    """Device failure (no GPU, launch error, out of memory)."""


_c_int, _c_double, _c_size, _c_long = ctypes.c_int, ctypes.c_double, ctypes.c_size_t, ctypes.c_long
_vp, _cp = ctypes.c_void_p, ctypes.c_char_p

# name -> (restype, argtypes); mirrors include/hmdp.h one to one
SIGNATURES = {
    "hmdp_last_error": (_cp, []),
    "hmdp_create": (_c_int, [_cp, _c_size, _c_int, _c_int, _c_int, ctypes.POINTER(_vp)]),
    "hmdp_destroy": (_c_int, [_vp]),
    "hmdp_model_validate": (_c_int, [_cp, _c_size]),
    "hmdp_model_info": (_c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_compute": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_compute_csr": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_double, _c_int, _c_int,
                                  _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_build_neighbors": (_c_int, [_vp, _c_int, _vp, _vp, _c_double, _c_int, _vp, _vp, _vp, _vp]),
    "hmdp_descriptors": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_switch_value": (_c_double, [_c_double, _c_double]),
    "hmdp_switch_derivative": (_c_double, [_c_double, _c_double]),
    "hmdp_counters": (_c_int, [_vp, _c_int, _c_int, ctypes.c_longlong, _c_int, _vp]),
    "hmdp_prepare": (_c_int, [_vp, _c_int, _vp, _c_int]),
    "hmdp_compute_device": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_check": (_c_int, [_vp]),
    "hmdp_kernels_per_eval": (_c_int, [_vp]),
    "hmdp_md_create": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_double, _c_int, _c_int,
                                ctypes.POINTER(_vp)]),
    "hmdp_md_run": (_c_int, [_vp, _c_int]),
    "hmdp_md_enqueue": (_c_int, [_vp, _c_int]),
    "hmdp_set_stream": (_c_int, [_vp, _vp]),
    "hmdp_dd_setup": (_c_int, [_vp, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_int]),
    "hmdp_dd_phase": (_c_int, [_vp, _c_int, _c_int]),
    "hmdp_dd_buffer": (_c_int, [_vp, _c_int, ctypes.POINTER(_vp)]),
    "hmdp_dd_result": (_c_int, [_vp, _vp, _vp, _vp]),
    "hmdp_profile": (_c_int, [_vp, _c_int]),
    "hmdp_profile_read": (_c_int, [_vp, _vp, _c_int, _vp]),
    "hmdp_profile_name": (_cp, [_vp, _c_int]),
    "hmdp_peak_fp32": (_c_int, [_c_int, _c_int, _vp]),
    "hmdp_peak_tf32x3": (_c_int, [_c_int, _c_int, _vp]),
    "hmdp_md_get": (_c_int, [_vp, _vp, _vp, _vp, _vp]),
    "hmdp_md_stats": (_c_int, [_vp, _vp, _vp]),
    "hmdp_md_destroy": (_c_int, [_vp]),
    "hmdp_compute_group": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _vp, _c_int, _vp, _vp,
                                    _vp, _vp]),
    "hmdp_make_model_json": (_c_long, [_c_int, _c_int, _c_double, _c_int, _c_int, _c_int,
                                       ctypes.c_uint64, _vp, _c_long]),
    "hmdp_gdd_setup": (_c_int, [_vp, _c_int, _vp, _vp, _vp, _c_int, _c_int]),
    "hmdp_gdd_bind": (_c_int, [_vp, _c_int, _vp]),
    "hmdp_gdd_phase": (_c_int, [_vp, _c_int, _c_int, _c_double]),
    "hmdp_gdd_counts": (_c_int, [_vp, _vp]),
    "hmdp_gdd_launches": (_c_int, [_vp, _vp]),
    "hmdp_gdd_set_mode": (_c_int, [_vp, _c_int]),
    "hmdp_tc_mlp": (_c_int, [_c_int, _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "hmdp_peak_tcgen05_tf32": (_c_int, [_c_int, _c_int, _vp]),
    "hmdp_nccl_unique_id": (_c_int, [_vp]),
    "hmdp_gdd_attach_nccl": (_c_int, [_vp, _vp, _c_int, _c_int]),
    "hmdp_gdd_hub_create": (_c_int, [_c_int, ctypes.POINTER(_vp)]),
    "hmdp_gdd_hub_destroy": (_c_int, [_vp]),
    "hmdp_gdd_attach_hub": (_c_int, [_vp, _vp]),
    "hmdp_gdd_attach_callback": (_c_int, [_vp, _vp, _vp]),
    "hmdp_gdd_plan": (_c_int, [_vp]),
    "hmdp_gdd_step": (_c_int, [_vp, _c_int, _c_double]),
    "hmdp_gdd_halo_stats": (_c_int, [_vp, _vp]),
    "hmdp_gdd_roles": (_c_int, [_vp, _vp]),
    "hmdp_ff_create": (_c_int, [_c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _c_int, _c_double,
                                _c_double, _c_double, _vp, _vp, _c_int, _vp, _vp, _c_int, _vp, _vp,
                                _c_int, _vp, _vp, ctypes.POINTER(_vp)]),
    "hmdp_ff_compute": (_c_int, [_vp, _vp, _vp, _c_int, _vp, _vp, _vp, _vp]),
    "hmdp_ff_destroy": (_c_int, [_vp]),
    "hmdp_hybrid_create": (_c_int, [_vp, _vp, _c_int, _vp, _c_int, _vp, _vp, _vp, _vp, _vp, _c_double,
                                    _c_int, _c_int, ctypes.POINTER(_vp)]),
    "hmdp_hybrid_run": (_c_int, [_vp, _c_int]),
    "hmdp_hybrid_get": (_c_int, [_vp, _vp, _vp, _vp, _vp]),
    "hmdp_hybrid_destroy": (_c_int, [_vp]),
    "hmdp_make_dp_model_json": (_c_long, [_c_int, _c_int, _c_double, _c_double, _c_int, _c_int,
                                          ctypes.c_uint64, _vp, _c_long]),
    "hmdp_synthetic_system": (_c_int, [_c_int, _c_double, _c_double, ctypes.c_uint64, _c_double,
                                       _vp, _vp, _vp, _vp, _vp]),
}

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load (building first if needed and nvcc is available) libhmdp.so."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import build as _build

            _build.build()
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhmdp.so missing at {LIB_PATH}; run paper_2602_02234_b200/build.py")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
        return _lib


def check(code: int) -> None:
    """Map a C-ABI return code to the reference's exception types."""
    if code == HMDP_OK:
        return
    msg = lib().hmdp_last_error().decode("utf-8", "replace")
    if code == HMDP_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if code == HMDP_RUNTIME_ERROR:
        raise RuntimeError(msg)  # std::runtime_error
    raise HmdpCudaError(msg)


def ptr(a) -> ctypes.c_void_p | None:
    """Data pointer of a numpy array (or None)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)

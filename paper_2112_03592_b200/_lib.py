"""ctypes binding of the C-ABI in include/aprgpu.h (libaprgpu.so).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import of the first entry point, loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libaprgpu.so")

OK, ERR_RANGE, ERR_CAPABILITY, ERR_INTEGRITY, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_INVALID = range(8)
HOST, DEVICE = 0, 1
PAD_ZERO, PAD_REFLECT = 0, 1
ACCUM_EXACT, ACCUM_FAST = 0, 1
PYR_RESTRICTED, PYR_RESCALED, PYR_UNIFORM, PYR_EXPLICIT = 0, 1, 2, 3
LEAF, TREE = 0, 1


class AccessDesc(C.Structure):
    _fields_ = [
        ("l_min", C.c_int32), ("l_max", C.c_int32),
        ("z_dim", C.c_void_p), ("x_dim", C.c_void_p), ("y_dim", C.c_void_p),
        ("y_idx", C.c_void_p), ("n_particles", C.c_uint64),
        ("xz_end", C.c_void_p), ("n_rows", C.c_uint64),
        ("level_offset", C.c_void_p),
    ]


class AccessInfo(C.Structure):
    _fields_ = [("l_min", C.c_int32), ("l_max", C.c_int32), ("n_particles", C.c_uint64), ("n_rows", C.c_uint64)]


_lib = None
_lock = threading.Lock()

class BuildParamsC(C.Structure):  # aprgpu_build_params
    _fields_ = [("rel_error", C.c_double), ("sigma_mode", C.c_int), ("sigma_value", C.c_double),
                ("sigma_window", C.c_int), ("sigma_floor", C.c_double), ("gradient_mode", C.c_int),
                ("smoothing_passes", C.c_int)]


class PatchSpecC(C.Structure):  # aprgpu_patch_spec
    _fields_ = [(n, C.c_int) for n in ("level", "z_begin", "z_end", "x_begin", "x_end", "pad", "pad_mode")]


_SIGS = {
    "aprgpu_init": [C.c_int, C.POINTER(C.c_void_p)],
    "aprgpu_ctx_free": [C.c_void_p],
    "aprgpu_ctx_stream": [C.c_void_p, C.POINTER(C.c_void_p)],
    "aprgpu_version": [],
    "aprgpu_upload_access": [C.c_void_p, C.POINTER(AccessDesc), C.POINTER(AccessDesc), C.c_void_p,
                             C.POINTER(C.c_void_p)],
    "aprgpu_apr_free": [C.c_void_p],
    "aprgpu_apr_dims": [C.c_void_p, C.c_void_p],
    "aprgpu_access_get_info": [C.c_void_p, C.c_int, C.POINTER(AccessInfo)],
    "aprgpu_apr_map_tiles": [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "aprgpu_apr_restrict": [C.c_void_p, C.c_int, C.c_int32, C.c_int32],
    "aprgpu_map_records": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p,
                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)],
    "aprgpu_download_access": [C.c_void_p, C.c_int] + [C.c_void_p] * 6,
    "aprgpu_row_index": [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                         C.POINTER(C.c_uint64)],
    "aprgpu_fill_tree": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p],
    "aprgpu_rebuild_index": [C.c_void_p, C.c_void_p],
    "aprgpu_restrict_stencil": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_gaussian_stencil": [C.c_double, C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_box_stencil": [C.c_int, C.c_void_p],
    "aprgpu_sobel_stencil": [C.c_int, C.c_void_p],
    "aprgpu_pyramid_create": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                              C.POINTER(C.c_void_p)],
    "aprgpu_pyramid_create_explicit": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                       C.POINTER(C.c_void_p)],
    "aprgpu_pyramid_free": [C.c_void_p],
    "aprgpu_pyramid_level": [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_convolve": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                        C.c_void_p],
    "aprgpu_rl": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                  C.c_void_p, C.c_int, C.c_void_p],
    "aprgpu_rl_resume": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                         C.c_double, C.c_int, C.c_void_p, C.c_int, C.c_void_p],
    "aprgpu_host_alloc": [C.c_uint64, C.POINTER(C.c_void_p)],
    "aprgpu_host_free": [C.c_void_p],
    "aprgpu_sequential_sum": [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.POINTER(C.c_double), C.c_void_p],
    "aprgpu_fill_tree_sums": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p],
    "aprgpu_tree_scratch": [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)],
    "aprgpu_fill_tree_finalize": [C.c_void_p, C.c_void_p, C.c_void_p],
    "aprgpu_multi_create": [C.c_void_p, C.c_int, C.POINTER(AccessDesc), C.POINTER(AccessDesc), C.c_void_p, C.c_int,
                            C.POINTER(C.c_void_p)],
    "aprgpu_multi_free": [C.c_void_p],
    "aprgpu_multi_info": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "aprgpu_multi_convolve": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_void_p],
    "aprgpu_convolve_slab_band": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_convolve_slab": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                             C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_tile_apr": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)],
    "aprgpu_tile_values": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p],
    "aprgpu_launch_count": [C.c_void_p, C.POINTER(C.c_uint64)],
    "aprgpu_generate_spheres": [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_void_p, C.c_int],
    "aprgpu_build_apr_params": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                C.POINTER(C.c_void_p)],
    "aprgpu_build_apr": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                         C.POINTER(C.c_void_p)],
    "aprgpu_apr_values": [C.c_void_p, C.c_void_p, C.c_int],
    "aprgpu_convolve_pixels": [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                               C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p],
    "aprgpu_load_apr": [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)],
    "aprgpu_save_apr": [C.c_void_p, C.c_char_p, C.c_void_p, C.c_int],
    "aprgpu_apr_params": [C.c_void_p, C.c_void_p],
    "aprgpu_validate_access": [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int), C.c_char_p, C.c_size_t],
    "aprgpu_reconstruct_level": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p],
    "aprgpu_reconstruct_patch": [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p],
}

EXPORTED = sorted(list(_SIGS) + ["aprgpu_last_error"])


def lib() -> C.CDLL:
    """Load libaprgpu.so (raises if it was not built -- there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"aprgpu CUDA library not built: {LIB_PATH} is missing (run `make lib` or "
                    "__graft_entry__.build()); the product path has no CPU fallback")
            L = C.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = C.c_int
            L.aprgpu_last_error.argtypes = []
            L.aprgpu_last_error.restype = C.c_char_p
            _lib = L
        return _lib


class AprError(RuntimeError):
    status = ERR_INVALID


def check(status: int) -> None:
    if status == OK:
        return
    from . import errors
    msg = lib().aprgpu_last_error().decode(errors="replace")
    raise errors.from_status(status, msg)

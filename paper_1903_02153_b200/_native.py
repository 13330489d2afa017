"""ctypes binding of libbfmm.so (the C ABI declared in include/bfmm.h).

The library is located in-tree (paper_1903_02153_b200/_lib/libbfmm.so,
built by ``python -m paper_1903_02153_b200.build``).  A missing library is
a hard error: the product has no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import NativeLibraryError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libbfmm.so")

_P = C.c_void_p
_I64 = C.c_int64
_I = C.c_int
_D = C.c_double
_SZ = C.c_size_t
_DP = C.POINTER(C.c_double)

# name -> (restype, argtypes); keep in sync with include/bfmm.h
SIGNATURES = {
    "bfmm_last_error": (C.c_char_p, []),
    "bfmm_version": (_I, []),
    "bfmm_tree_scratch_bytes": (_SZ, [_I64, _I]),
    "bfmm_tree_build": (_I, [_P, _I64, _DP, _I, _P, _SZ, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "bfmm_gather_weights": (_I, [_P, _I64, _I, _P, _P, _P, _P, _P]),
    "bfmm_p2m": (_I, [_P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _DP, _DP, _P, _P, _P]),
    "bfmm_p2m_cells": (_I, [_P, _P, _I, _P, _P, _I, _I, _I, _DP, _DP, _P, _P, _P]),
    "bfmm_l2p_cells": (_I, [_P, _I, _P, _P, _I, _I, _I, _DP, _DP, _P, _P, _P, _P]),
    "bfmm_p2m_pair": (_I, [_P, _P, _P, _P, _I, _I, _I, _DP, _DP, _P, _P, _P, _P]),
    "bfmm_l2p_pair": (_I, [_P, _P, _P, _I, _I, _I, _DP, _DP, _P, _P, _P, _P, _P]),
    "bfmm_p2m_sparse": (_I, [_P, _P, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _DP, _DP, _P, _P, _P]),
    "bfmm_m2m": (_I, [_P, _P, _I64, _I, _I, _DP, _P]),
    "bfmm_rows_gemm": (_I, [_P, _I64, _I, _P, _I, _P, _D, _D, _I, _P]),
    "bfmm_rows_gemm_i8": (_I, [_P, _I64, _I, _P, _P, _I, _P, _D, _P, _P]),
    "bfmm_rows_gemm_max": (_I, [_P, _I64, _I, _P, _I, _P, _D, _P, _P]),
    "bfmm_rows_gemm_scatter": (_I, [_P, _I64, _I, _P, _I, _P, _D, _D, _I, _P, _I64, _P]),
    "bfmm_rows_gemm_cells": (_I, [_P, _I64, _I, _P, _I, _P, _D, _P, _I64, _P]),
    "bfmm_m2l_cheb_cells": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P]),
    "bfmm_octant_histogram": (_I, [_P, _P, _I64, _P, _P]),
    "bfmm_group_by_octant_scratch_bytes": (_SZ, [_I64]),
    "bfmm_group_by_octant": (_I, [_P, _I64, _P, _P, _SZ, _P]),
    "bfmm_active_cells_scratch_bytes": (_SZ, [_I64]),
    "bfmm_active_cells": (_I, [_P, _P, _I64, _I, _I64, _I64, _P, _SZ, _P, _P, _P]),
    "bfmm_m2l_cheb_splits": (_I, [_I, _I, _I, _I64]),
    "bfmm_m2l_cheb": (_I, [_P, _P, _I, _I, _I, _I, _I64, _I64, _P, _P]),
    "bfmm_m2l_i8_zs_bytes": (_SZ, [_I64, _I, _I]),
    "bfmm_m2l_i8_slice_z": (_I, [_P, _I64, _I, _I, _I, _P, _P, _P]),
    "bfmm_m2l_i8_slice_z_cells": (_I, [_P, _I64, _I, _I, _I, _P, _P, _P, _P]),
    "bfmm_m2l_i8_zmax": (_I, [_P, _I64, _I, _I, _P, _P]),
    "bfmm_m2l_i8_splits": (_I, [_I, _I, _I, _I64]),
    "bfmm_m2l_i8": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I64, _I64, _P]),
    "bfmm_m2l_i8_cells": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "bfmm_device_dmma_probe": (_I, [_DP, _P]),
    "bfmm_device_i8_probe": (_I, [_DP, _P]),
    "bfmm_device_i8_probe_n": (_I, [_I, _DP, _P]),
    "bfmm_tc_i8_selftest": (_I, [_P, _P, _I, _P, _P]),
    "bfmm_device_dmma_sweep": (_I, [_I, _I, _DP, _P]),
    "bfmm_launch_count": (C.c_longlong, []),
    "bfmm_m2l_fft_scratch_bytes": (_I, [_I, _I, _I, C.POINTER(_SZ)]),
    "bfmm_m2l_fft": (_I, [_P, _P, _I, _I, _I, _P, _D, _I64, _I64, _P, _SZ, _P]),
    "bfmm_l2l": (_I, [_P, _P, _I64, _I, _I, _DP, _P]),
    "bfmm_l2p": (_I, [_P, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _DP, _DP, _P, _P, _P, _P]),
    "bfmm_l2p_points": (_I, [_P, _I, _P, _P, _P, _P, _I64, _I, _I, _I, _DP, _DP, _P, _P, _P, _P]),
    "bfmm_kernel_compile": (_I, [_I, C.c_char_p, C.POINTER(_I)]),
    "bfmm_p2p_scratch_bytes": (_SZ, [_I64, _I64]),
    "bfmm_p2p": (_I, [_I, _P, _P, _P, _P, _P, _I64, _P, _P, _I, _P, _P, _I, _I64, _I64, _P, _P,
                      _SZ, _P]),
    "bfmm_p2p_cells": (_I, [_I, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _P, _I, _P, _P, _I, _I64,
                            _I64, _P, _P, _SZ, _P]),
    "bfmm_p2p_grouped": (_I, [_I, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _I, _I64, _I64, _P, _P]),
    "bfmm_p2p_symmetric_scratch_bytes": (_SZ, [_I64, _I64]),
    "bfmm_p2p_symmetric": (_I, [_I, _P, _P, _P, _P, _P, _I64, _P, _P, _I, _I64, _I64, _I64, _D,
                                _P, _P, _SZ, _P]),
    "bfmm_direct": (_I, [_I, _P, _I64, _P, _P, _I64, _I, _P, _P]),
    "bfmm_kernel_block": (_I, [_I, _P, _I64, _P, _I64, _P, _I, _P, _P, _P]),
    "bfmm_p2p_locate": (_I, [_I, _P, _P, _P, _P, _P, _I64, _P, _P, _P, _I, _P, _P]),
    "bfmm_scatter_output": (_I, [_P, _P, _P, _I64, _I, _P, _P, _P]),
    "bfmm_far_pairs": (_I, [_I, _I, _P, _P, _P, _P, _SZ, _P]),
    "bfmm_far_pairs_scratch_bytes": (_SZ, [_I]),
    "bfmm_near_pairs": (_I, [_I, _I, _P, _P, _I64, _P, _P, _P, _P]),
    "bfmm_near_pair_count": (_I, [_P, _P, _P, _I64, _P, _I, _P, _P]),
    "bfmm_level2_work": (_I, [_P, _P, _P, _I64, _P, _I, _P, _P]),
    "bfmm_device_fp64_probe": (_I, [_DP, _P]),
}

#: bfmm_m2l_i8* S flag: 8-bit digits (include/bfmm.h BFMM_I8_BASE256)
I8_BASE256 = 0x100
#: bfmm_m2l_i8_slice_z S flag: zmax given (include/bfmm.h BFMM_I8_ZMAX_GIVEN)
I8_ZMAX_GIVEN = 0x200

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load libbfmm.so once and attach the signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} is missing; build it with `python -m paper_1903_02153_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().bfmm_last_error().decode(errors="replace")
        raise NativeLibraryError(f"{what} failed ({rc}): {msg}")


def dptr(arr):
    """Host float64 numpy array -> ctypes double pointer (keeps no reference)."""
    return arr.ctypes.data_as(_DP)

"""ctypes binding of libnufft_b200.so (the C-ABI in include/nufft_b200.h).

Loading fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# NUFFT_B200_LIB: load another build of the library (A/B measurements of two builds)
LIB_PATH = os.environ.get("NUFFT_B200_LIB") or os.path.join(HERE, "libnufft_b200.so")

_sz = C.c_size_t
_vp = C.c_void_p
_dp = C.POINTER(C.c_double)
_i = C.c_int


class PlanInfo(C.Structure):
    _fields_ = [
        ("n", _sz), ("rank", _sz), ("rank2", _sz), ("effective_rank", _sz),
        ("gamma", C.c_double), ("gamma2", C.c_double), ("epsilon", C.c_double),
        ("btrivial", _i), ("m", _sz), ("ncols", _sz), ("device", _i), ("path", _i),
    ]


class CgReport(C.Structure):
    _fields_ = [("iterations", _sz), ("relative_residual", C.c_double), ("converged", _i),
                ("history_len", _sz)]


_SIGS = {
    "nufft_last_error": (C.c_char_p, []),
    "nufft_abi_version": (_i, []),
    "nufft_device_count": (_i, [C.POINTER(_i)]),
    "nufft_lambert_w": (_i, [C.c_double, _dp]),
    "nufft_bessel_j_int": (_i, [_i, C.c_double, _dp]),
    "nufft_bessel_j_signed": (_i, [_i, C.c_double, _dp]),
    "nufft_select_rank": (_i, [C.c_double, C.c_double, C.POINTER(_sz)]),
    "nufft_cheb_coefficients": (_i, [C.c_double, _sz, _vp]),
    "nufft_cheb_eval_matrix": (_i, [_vp, _sz, _sz, _vp]),
    "nufft_build_factors": (_i, [_vp, _sz, C.c_double, _vp, _sz, C.c_double, C.POINTER(_sz), _vp, _vp]),
    "nufft_fft_forward_host": (_i, [_vp, _vp, _sz]),
    "nufft_fft_inverse_host": (_i, [_vp, _vp, _sz]),
    "nufft_fft_2d_forward_host": (_i, [_vp, _vp, _sz, _sz]),
    "nufft_fft_cols_forward_host": (_i, [_vp, _sz, _sz]),
    "nufft_fft_rows_forward_host": (_i, [_vp, _sz, _sz]),
    "nufft_fft_exec": (_i, [_vp, _vp, _sz, _sz, _i, _vp]),
    "nufft_fft_exec_count": (C.c_uint64, [_sz]),
    "nufft_fft_reset_exec_counts": (None, []),
    "nufft_kernel_launch_count": (C.c_uint64, []),
    "nufft_normalize_samples": (_i, [_vp, _sz, _vp]),
    "nufft_grid_assign": (_i, [_vp, _sz, _sz, _vp, _vp, _dp]),
    "nufft_plan2_create": (_i, [_vp, _sz, C.c_double, _i, C.POINTER(_vp)]),
    "nufft_plan2_create_device": (_i, [_vp, _sz, C.c_double, _i, C.POINTER(_vp)]),
    "nufft_plan2_destroy": (None, [_vp]),
    "nufft_plan2_info": (_i, [_vp, C.POINTER(PlanInfo)]),
    "nufft_plan2_samples": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_plan2_factors": (_i, [_vp, _vp, _vp]),
    "nufft_plan2_exec": (_i, [_vp, _vp, _vp, _sz, _vp]),
    "nufft_plan2_exec_terms": (_i, [_vp, _vp, _vp, _sz, _sz, _sz, _vp]),
    "nufft_plan2_exec_host": (_i, [_vp, _vp, _sz, _vp, _sz]),
    "nufft_plan2_exec_timed": (_i, [_vp, _vp, _vp, _vp, _i]),
    "nufft_plan2_timing_read": (_i, [_vp, _i, _dp, _dp]),
    "nufft_plan2_adjoint": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_plan2_adjoint_host": (_i, [_vp, _vp, _sz, _vp]),
    "nufft_plan1_create": (_i, [_vp, _sz, C.c_double, _i, C.POINTER(_vp)]),
    "nufft_plan1_destroy": (None, [_vp]),
    "nufft_plan1_info": (_i, [_vp, C.POINTER(PlanInfo)]),
    "nufft_plan1_samples": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_plan1_exec": (_i, [_vp, _vp, _vp, _sz, _vp]),
    "nufft_plan1_exec_host": (_i, [_vp, _vp, _sz, _vp, _sz]),
    "nufft_plan1_adjoint": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_plan1_adjoint_host": (_i, [_vp, _vp, _sz, _vp]),
    "nufft_toeplitz_from_first_column": (_i, [_vp, _sz, _i, C.POINTER(_vp)]),
    "nufft_toeplitz_from_normal": (_i, [_vp, C.POINTER(_vp)]),
    "nufft_toeplitz_from_gram": (_i, [_vp, C.POINTER(_vp)]),
    "nufft_toeplitz_destroy": (None, [_vp]),
    "nufft_toeplitz_size": (_i, [_vp, C.POINTER(_sz)]),
    "nufft_toeplitz_members": (_i, [_vp, _vp, _vp]),
    "nufft_toeplitz_matvec": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_toeplitz_matvec_host": (_i, [_vp, _vp, _sz, _vp]),
    "nufft_cg_toeplitz_host": (_i, [_vp, _vp, _sz, C.c_double, _sz, _vp, C.POINTER(CgReport), _vp, _sz]),
    "nufft_inufft2_host": (_i, [_vp, _vp, _vp, _sz, C.c_double, _vp, C.POINTER(CgReport), _vp, _sz]),
    "nufft_inufft2": (_i, [_vp, _vp, _vp, C.c_double, _vp, C.POINTER(CgReport), _vp]),
    "nufft_inufft1_host": (_i, [_vp, _vp, _vp, _sz, C.c_double, _vp, C.POINTER(CgReport), _vp, _sz]),
    "nufft_default_cg_max_iter": (_sz, [_sz]),
    "nufft_nudft_direct_host": (_i, [_vp, _sz, _vp, _vp, _sz, _vp, _i]),
    "nufft_nudft_direct": (_i, [_vp, _sz, _vp, _vp, _sz, _vp, _vp]),
    "nufft_nudft2d_direct_host": (_i, [_vp, _vp, _sz, _vp, _sz, _sz, _vp, _i]),
    "nufft_plan3_create": (_i, [_vp, _vp, _sz, _sz, C.c_double, _i, C.POINTER(_vp)]),
    "nufft_plan3_destroy": (None, [_vp]),
    "nufft_plan3_info": (_i, [_vp, C.POINTER(PlanInfo)]),
    "nufft_plan3_samples": (_i, [_vp, _vp, _vp, _vp]),
    "nufft_plan3_exec": (_i, [_vp, _vp, _vp, _sz, _vp]),
    "nufft_plan3_exec_host": (_i, [_vp, _vp, _sz, _vp, _sz]),
    "nufft_plan2d2_create": (_i, [_vp, _vp, _sz, _sz, _sz, _sz, C.c_double, _i, C.POINTER(_vp)]),
    "nufft_plan2d2_destroy": (None, [_vp]),
    "nufft_plan2d2_info": (_i, [_vp, C.POINTER(PlanInfo)]),
    "nufft_plan2d2_samples": (_i, [_vp] * 8),
    "nufft_plan2d2_exec": (_i, [_vp, _vp, _vp, _sz, _vp]),
    "nufft_plan2d2_exec_host": (_i, [_vp, _vp, _sz, _sz, _vp, _sz]),
    "nufft_plan2d2_exec_host_impl": (_i, [_vp, _vp, _sz, _sz, _vp, _sz, _i]),
    "nufft_comm_unique_id": (_i, [_vp]),
    "nufft_comm_init": (_i, [_vp, _i, _i, _i, C.POINTER(_vp)]),
    "nufft_comm_wrap": (_i, [_vp, _i, C.POINTER(_vp)]),
    "nufft_comm_destroy": (None, [_vp]),
    "nufft_comm_info": (_i, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "nufft_multi_term_range": (_i, [_sz, _i, _i, C.POINTER(_sz), C.POINTER(_sz)]),
    "nufft_plan2_exec_multi": (_i, [_vp, _vp, _vp, _sz, _vp, _i, _i, _vp]),
    "nufft_plan2_exec_multi_host": (_i, [_vp, _vp, _sz, _vp, _sz, _vp, _i, _i]),
    "nufft_plan1_exec_terms": (_i, [_vp, _vp, _vp, _sz, _sz, _sz, _vp]),
    "nufft_plan1_exec_multi": (_i, [_vp, _vp, _vp, _sz, _vp, _i, _i, _vp]),
    "nufft_plan3_exec_terms": (_i, [_vp, _vp, _vp, _sz, _sz, _sz, _vp]),
    "nufft_plan3_exec_multi": (_i, [_vp, _vp, _vp, _sz, _vp, _i, _i, _vp]),
    "nufft_plan2d2_exec_terms": (_i, [_vp, _vp, _vp, _sz, _sz, _sz, _vp]),
    "nufft_plan2d2_exec_multi": (_i, [_vp, _vp, _vp, _sz, _vp, _i, _i, _vp]),
    "nufft_plan2_exec_terms_sorted": (_i, [_vp, _vp, _vp, _sz, _sz, _vp]),
    "nufft_plan2_reduce_chunks": (_i, [_vp, _i, _vp]),
    "nufft_plan2_unpermute": (_i, [_vp, _vp, _vp, _sz, _vp]),
    "nufft_sampler_create": (_i, [C.c_uint64, C.POINTER(_vp)]),
    "nufft_sampler_destroy": (None, [_vp]),
    "nufft_sampler_normal": (C.c_double, [_vp]),
    "nufft_sampler_uniform": (C.c_double, [_vp]),
    "nufft_sampler_uniform_vector": (_i, [_vp, _sz, C.c_double, C.c_double, _vp]),
    "nufft_sampler_complex_vector": (_i, [_vp, _sz, _vp]),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


_lib = None


def lib() -> C.CDLL:
    """Load the CUDA library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing — build it with paper_1701_04492_b200.build_ext.build() "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib

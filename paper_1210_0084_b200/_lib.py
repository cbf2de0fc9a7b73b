"""ctypes declarations of libslicq.so (include/slicq.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLICQ_LIB", os.path.join(_HERE, "libslicq.so"))

SLICQ_OK = 0
ERRORS = {-1: "EINVAL", -2: "ENOTFRAME", -3: "ESHAPE", -4: "ECUDA", -5: "ENOMEM",
          -6: "EINTERNAL", -7: "EUNSUPPORTED"}
PLAN_HOST_ONLY = 1
WINDOWS = {"hann": 0, "blackman_harris": 1}

# every symbol include/slicq.h declares, with (restype, argtypes)
_p, _i64, _i32, _d, _sz, _u = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.c_size_t, C.c_uint
SIGNATURES = {
    "plan_create": (_i32, [_d, _d, _d, _i32, _i64, _i64, _i32, C.POINTER(_p)]),
    "plan_create_ex": (_i32, [_d, _d, _d, _i32, _i64, _i64, _i32, _u, C.POINTER(_p)]),
    "plan_create_ex2": (_i32, [_d, _d, _d, _i32, _i64, _i64, _i32, _u, _i32, _d, _i64,
                               C.POINTER(_p)]),
    "slicq_approx_error": (_i32, [_p, _p, _p, _p, _i64, _p, _p]),
    "slicq_coeffs_per_slice_full": (_i64, [_p]),
    "slicq_workspace_bytes_complex": (_sz, [_p, _i64, _i64, _i64]),
    "slicq_forward_complex": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_inverse_complex": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_nsgt_forward_complex": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_nsgt_inverse_complex": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_approx_error_complex": (_i32, [_p, _p, _p, _p, _i64, _p, _p]),
    "slicq_apply_mask": (_i32, [_p, _p, _p, _i64, _i32, _i32, _p]),
    "slicq_spectrogram": (_i32, [_p, _p, _i64, _i64, _p, _p]),
    "slicq_transpose_bins": (_i32, [_p, _p, _p, _i64, _i32, _p]),
    "plan_destroy": (None, [_p]),
    "slicq_num_channels": (_i32, [_p]),
    "slicq_num_cq_channels": (_i32, [_p]),
    "slicq_channel_lengths": (_i32, [_p, _p]),
    "slicq_channel_offsets": (_i32, [_p, _p]),
    "slicq_coeffs_per_slice": (_i64, [_p]),
    "slicq_sl_len": (_i64, [_p]),
    "slicq_padded_length": (_i64, [_p, _i64]),
    "slicq_num_slices": (_i64, [_p, _i64]),
    "slicq_halo": (_i64, [_p]),
    "slicq_workspace_bytes": (_sz, [_p, _i64, _i64]),
    "slicq_kernel_launches": (_i32, [_p, _i32, _i64, _i64]),
    "slicq_nsgt_forward": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_nsgt_inverse": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_inverse_masked": (_i32, [_p, _p, _p, _i32, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_process_host_workspace_bytes": (_sz, [_p, _i64, _i64, _i32]),
    "slicq_process_host": (_i32, [_p, _p, _p, _i64, _i64, _i32, _p, _p, _p, _sz, _p]),
    "slicq_plan_export": (_i32, [_p, _p, _p, _p, _p, _p, _p, _p]),
    "slicq_filter_total_length": (_i64, [_p]),
    "slicq_last_error": (C.c_char_p, []),
    "slicq_forward": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_inverse": (_i32, [_p, _p, _i64, _i64, _p, _p, _sz, _p]),
    "slicq_forward_range": (_i32, [_p, _p, _i64, _i64, _i64, _i64, _i64, _i64, _i64, _p, _p,
                                   _sz, _p]),
    "slicq_inverse_range": (_i32, [_p, _p, _i64, _i64, _i64, _i64, _p, _i64, _p, _i64, _p, _sz,
                                   _p]),
    "slicq_overlap_add": (_i32, [_p, _i64, _p, _i64, _i64, _p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libslicq.so; raises loudly if it is missing (there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libslicq.so not built ({LIB_PATH}); run "
                              "`python -m paper_1210_0084_b200.build` — there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class SlicqError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().slicq_last_error().decode(errors="replace")
        super().__init__(f"{where}: SLICQ_{ERRORS.get(code, code)}: {msg}")
        self.code = code


def check(rc: int, where: str) -> int:
    if rc < 0:
        raise SlicqError(rc, where)
    return rc

# slicq_coeff_fn(user, coeffs, slice0, nslices, batch, stream) -> int
COEFF_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p)

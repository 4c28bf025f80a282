"""ctypes declarations of the C-ABI in include/lyapgpu.h (argument marshalling only).

The shared library is built in-tree (paper_2312_08201_b200/liblyapgpu.so, see build.py).  There
is no fallback: if it is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import pathlib

LIB_PATH = pathlib.Path(__file__).resolve().parent / "liblyapgpu.so"

LYAP_OK, LYAP_EINVAL, LYAP_ENOMEM, LYAP_ECUDA, LYAP_EEIG, LYAP_ESINGULAR, LYAP_EPARTIAL, LYAP_ENODEV = range(8)
STATUS_NAMES = {0: "LYAP_OK", 1: "LYAP_EINVAL", 2: "LYAP_ENOMEM", 3: "LYAP_ECUDA", 4: "LYAP_EEIG",
                5: "LYAP_ESINGULAR", 6: "LYAP_EPARTIAL", 7: "LYAP_ENODEV"}
LYAP_KMAX = 8

# every symbol include/lyapgpu.h declares (checked by tests/test_abi.py)
EXPORTED = ("lyap_default_opts", "lyap_setup", "lyap_trace_batch", "lyap_trace_batch_ex", "lyap_trace_batch_x",
            "lyap_stable_batch", "lyap_setup_qlin", "lyap_ek_trace_batch_ex",
            "lyap_get_info",
            "lyap_get_stats", "lyap_reset_stats", "lyap_apply_C", "lyap_apply_C_mixed", "lyap_export_state", "lyap_destroy",
            "lyap_last_error", "lyap_solution", "lyap_setup_like", "lyap_set_recycle",
            "lyap_build_recycle", "lyap_ek_setup", "lyap_ek_trace_batch", "lyap_ek_destroy", "lyap_ek_last_error")


class Opts(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_dim", C.c_int32), ("max_restarts", C.c_int32),
                ("batch", C.c_int32), ("warm_start", C.c_int32), ("max_cond_S", C.c_double),
                ("device", C.c_int32), ("profile", C.c_int32), ("schedule", C.c_int32), ("recycle", C.c_int32),
                ("check_stable", C.c_int32), ("coarse", C.c_int32), ("mixed", C.c_int32),
                ("mixed_eta", C.c_double)]


class Info(C.Structure):
    _fields_ = [("n", C.c_int64), ("k", C.c_int64), ("npad", C.c_int64), ("n_pairs", C.c_int64),
                ("t0", C.c_double), ("cond_S", C.c_double), ("min_lam_sum", C.c_double),
                ("max_abs_lam", C.c_double), ("setup_ms", C.c_double), ("batch", C.c_int32),
                ("max_dim", C.c_int32), ("wcost", C.c_double * LYAP_KMAX), ("coarse", C.c_int32),
                ("coarse_build_ms", C.c_double), ("mixed_mode", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("k1_launches", C.c_int64), ("k1_vectors", C.c_int64), ("k1_ms", C.c_double),
                ("k1_flops", C.c_double), ("iterations", C.c_int64), ("kernel_launches", C.c_int64),
                ("batch_ms", C.c_double), ("recycle_build_ms", C.c_double),
                ("graph_instantiations", C.c_int64), ("graph_updates", C.c_int64),
                ("k1_exact_vectors", C.c_int64)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is not built; run `python paper_2312_08201_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    P = C.c_void_p
    dp = C.POINTER(C.c_double)
    lib.lyap_default_opts.argtypes = [C.POINTER(Opts)]
    lib.lyap_default_opts.restype = None
    lib.lyap_setup.argtypes = [C.c_int64, C.c_int64, dp, dp, dp, dp, dp, C.POINTER(Opts), C.POINTER(P)]
    lib.lyap_setup.restype = C.c_int
    lib.lyap_trace_batch.argtypes = [P, C.c_int64, P, P, P, C.c_int, P]
    lib.lyap_trace_batch.restype = C.c_int
    lib.lyap_trace_batch_ex.argtypes = [P, C.c_int64, P, P, P, P, P, C.c_int, P]
    lib.lyap_trace_batch_ex.restype = C.c_int
    lib.lyap_trace_batch_x.argtypes = [P, C.c_int64, P, P, P, P, P, P, P, P]
    lib.lyap_trace_batch_x.restype = C.c_int
    lib.lyap_ek_trace_batch_ex.argtypes = [P, C.c_int64, P, C.c_double, C.c_int32, P, P, P]
    lib.lyap_ek_trace_batch_ex.restype = C.c_int
    lib.lyap_setup_qlin.argtypes = [C.c_int64, C.c_int64, dp, dp, dp, dp, dp, C.POINTER(Opts), C.POINTER(P)]
    lib.lyap_setup_qlin.restype = C.c_int
    lib.lyap_stable_batch.argtypes = [P, C.c_int64, P, P, C.c_int, P]
    lib.lyap_stable_batch.restype = C.c_int
    lib.lyap_get_info.argtypes = [P, C.POINTER(Info)]
    lib.lyap_get_info.restype = C.c_int
    lib.lyap_get_stats.argtypes = [P, C.POINTER(Stats)]
    lib.lyap_get_stats.restype = C.c_int
    lib.lyap_reset_stats.argtypes = [P]
    lib.lyap_reset_stats.restype = C.c_int
    lib.lyap_apply_C.argtypes = [P, C.c_int64, P, P, P, P]
    lib.lyap_apply_C.restype = C.c_int
    lib.lyap_apply_C_mixed.argtypes = [P, C.c_int64, P, P, P, P]
    lib.lyap_apply_C_mixed.restype = C.c_int
    lib.lyap_export_state.argtypes = [P, P, P, P, P, P, P]
    lib.lyap_export_state.restype = C.c_int
    lib.lyap_setup_like.argtypes = [P, C.c_int64, dp, dp, C.POINTER(Opts), C.POINTER(P)]
    lib.lyap_setup_like.restype = C.c_int
    lib.lyap_ek_setup.argtypes = [C.c_int64, C.c_int64, dp, dp, dp, dp, dp, C.c_double, C.c_int32, C.POINTER(P)]
    lib.lyap_ek_setup.restype = C.c_int
    lib.lyap_ek_trace_batch.argtypes = [P, C.c_int64, P, C.c_double, C.c_int32, P, P, P]
    lib.lyap_ek_trace_batch.restype = C.c_int
    lib.lyap_ek_destroy.argtypes = [P]
    lib.lyap_ek_destroy.restype = None
    lib.lyap_ek_last_error.argtypes = [P]
    lib.lyap_ek_last_error.restype = C.c_char_p
    lib.lyap_build_recycle.argtypes = [P, C.c_int32, P, C.c_int32]
    lib.lyap_build_recycle.restype = C.c_int
    lib.lyap_set_recycle.argtypes = [P, C.c_int32, C.c_int32, P, P]
    lib.lyap_set_recycle.restype = C.c_int
    lib.lyap_solution.argtypes = [P, C.c_int64, P, P, P]
    lib.lyap_solution.restype = C.c_int
    lib.lyap_destroy.argtypes = [P]
    lib.lyap_destroy.restype = None
    lib.lyap_last_error.argtypes = [P]
    lib.lyap_last_error.restype = C.c_char_p
    return lib


lib = _load()


class LyapError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code

"""CPU checks of the C-ABI boundary: the library loads, exports every symbol include/lyapgpu.h
declares, and fails loudly (LYAP_ENODEV / LyapError) without a GPU instead of computing on the CPU."""
import ctypes as C
import pathlib
import re

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "lyapgpu.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lyap_[A-Za-z_0-9]+)\s*\(", text)))


def test_header_declares_expected_calls():
    names = declared_functions()
    for must in ("lyap_setup", "lyap_trace_batch", "lyap_destroy", "lyap_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2312_08201_b200 import EXPORTED, lib
    names = declared_functions()
    assert sorted(EXPORTED) == names
    raw = C.CDLL(str(ROOT / "paper_2312_08201_b200" / "liblyapgpu.so"))
    for nm in names:
        assert hasattr(raw, nm), nm
        assert getattr(lib, nm) is not None


def test_default_opts():
    from paper_2312_08201_b200 import default_opts
    o = default_opts()
    assert o.tol == 1e-12 and o.warm_start == 0 and o.max_restarts == 30 and o.max_cond_S == 1e8


def test_invalid_args_rejected_before_device():
    from paper_2312_08201_b200 import lib
    ctx = C.c_void_p()
    z = np.zeros(4)
    dp = z.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.lyap_setup(2, 0, dp, dp, dp, dp, dp, None, C.byref(ctx)) == 1  # k = 0
    assert lib.lyap_setup(2, 9, dp, dp, dp, dp, dp, None, C.byref(ctx)) == 1  # k > KMAX
    assert b"invalid" in lib.lyap_last_error(None)
    assert lib.lyap_trace_batch(None, 1, None, None, None, 0, None) == 1


def test_asymmetric_Q_rejected():
    """Q must be symmetric (the nk reduction needs it): LYAP_EINVAL, checked on the
    host before any device work."""
    from paper_2312_08201_b200 import LyapError, Problem
    Q = np.array([[1.0, 0.5], [0.0, 1.0]])
    with pytest.raises(LyapError) as ei:
        Problem(-np.eye(2), np.ones((2, 1)), np.ones((2, 1)), Q, np.eye(2))
    assert ei.value.code == 1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2312_08201_b200 import LyapError, Problem
    A0 = -np.eye(2)
    B = np.ones((2, 1))
    with pytest.raises(LyapError) as ei:
        Problem(A0, B, B, np.eye(2), np.eye(2))
    assert ei.value.code == 7  # LYAP_ENODEV


def test_product_package_does_not_import_oracle():
    """The product path never imports oracle/ (the CPU oracle is test infrastructure only)."""
    for p in (ROOT / "paper_2312_08201_b200").rglob("*.py"):
        src = p.read_text()
        assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), p

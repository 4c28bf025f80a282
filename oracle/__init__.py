"""CPU oracle for trace(E X(v)) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product path (paper_2312_08201_b200) never does.
"""
from .bartels_stewart import LEAF, form_A, lyap, sylvester_quasi_triangular, trace_batch, trace_EX
from .stability import rightmost_real_part, stable_mask, unstable_count

__all__ = ["LEAF", "form_A", "lyap", "sylvester_quasi_triangular", "trace_batch", "trace_EX",
           "rightmost_real_part", "stable_mask", "unstable_count"]

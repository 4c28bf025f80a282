"""CPU oracle of the stability filter (NEXT row f4) — TEST INFRASTRUCTURE ONLY.

Only tests/ may import it (the product path never does, and shares no code with it).

What it computes (Example 2): "we have computed the rightmost eigenvalue lambda of
A(v) and discarded those configurations for which Re(lambda) >= 0".  For each parameter vector v:

  1. form A(v) = A0 - Bl diag(v) Br^T explicitly (eq:formA);
  2. all eigenvalues of A(v) by LAPACK dgeev (numpy.linalg.eigvals);
  3. the rightmost one: max Re lambda;
  4. v is kept (stable) iff that real part is < 0.

Pins (tests/test_oracle_pins.py): the 1-DOF oscillator closed form (eigenvalues of
[[0, w], [-w, -c]]: Re = -c/2 for c < 2w, (-c + sqrt(c^2 - 4 w^2))/2 above; stable iff c > 0), a
diagonal seed with a rank-one update on one coordinate (the eigenvalues are the updated diagonal),
and the quadratic formula on random 2 x 2 instances.
"""
from __future__ import annotations

import numpy as np

from .bartels_stewart import form_A

__all__ = ["rightmost_real_part", "stable_mask", "unstable_count"]


def rightmost_real_part(A0, Bl, Br, v) -> float:
    """max Re lambda(A(v))."""
    return float(np.max(np.linalg.eigvals(form_A(A0, Bl, Br, v)).real))


def stable_mask(A0, Bl, Br, V) -> np.ndarray:
    """Boolean per row of V: A(v) stable (rightmost eigenvalue strictly in the left half-plane)."""
    V = np.atleast_2d(np.asarray(V, dtype=np.float64))
    return np.array([rightmost_real_part(A0, Bl, Br, v) < 0.0 for v in V], dtype=bool)


def unstable_count(A0, Bl, Br, v) -> int:
    """Number of eigenvalues of A(v) with Re > 0 (steps 1-2 above, then a count)."""
    return int(np.sum(np.linalg.eigvals(form_A(A0, Bl, Br, v)).real > 0.0))

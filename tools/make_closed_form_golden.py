"""Write tests/golden/one_dof.json and spec_examples.json from hand-derived closed forms.

1-DOF damped oscillator in modal phase-space form (PAPER.md:816-834 with BASELINE's -2*alpha*Omega),
one damper with modal weight phi:  A = [[0, w], [-w, -c]],  c = 2*alpha*w + v*phi^2,  Q = I.
Writing X = [[x, y], [y, z]], the three scalar equations of A X + X A^T = -I are
   (1,1): 2 w y = -1            -> y = -1/(2w)
   (2,2): -2 w y - 2 c z = -1   -> z = 1/c
   (1,2): w z - w x - c y = 0   -> x = 1/c + c/(2 w^2)
so trace X = 2/c + c/(2 w^2).  (The paper's printed X0 (1,1) block (3 alpha/2) Omega^-1,
PAPER.md:853-858, does not satisfy the (1,2) equation; reading R1.)

SPEC.md worked examples: diagonal A gives X_ij = -Q_ij/(a_i+a_j).
No oracle/ or product code is used here.
"""
import json
import pathlib

out = pathlib.Path(__file__).resolve().parents[1] / "tests" / "golden"
cases = []
for (w, a, phi, v) in [(1.0, 0.02, 1.0, 0.1), (1.0, 0.02, 1.0, 1.0), (1.0, 0.02, 1.0, 10.0),
                       (3.7, 0.005, 0.4, 2.5), (0.07, 0.01, 0.02, 1000.0), (12.0, 0.3, 2.0, 0.001)]:
    c = 2 * a * w + v * phi * phi
    cases.append({"omega": w, "alpha": a, "phi": phi, "v": v, "c": c,
                  "trace": 2.0 / c + c / (2.0 * w * w)})
(out / "one_dof.json").write_text(json.dumps({
    "source": "hand derivation in tools/make_closed_form_golden.py (DESIGN.md R1)",
    "cases": cases}, indent=1))

spec = {
    "source": "SPEC.md:74-75 (solve_lyap_dense examples), SPEC.md:165/201/210/219 (n=2 worked problem)",
    "lyap": [
        {"A": [[-1.0, 0.0], [0.0, -1.0]], "Q": [[1.0, 0.0], [0.0, 1.0]], "X": [[0.5, 0.0], [0.0, 0.5]]},
        {"A": [[-1.0, 0.0], [0.0, -2.0]], "Q": [[1.0, 1.0], [1.0, 1.0]],
         "X": [[0.5, 1.0 / 3.0], [1.0 / 3.0, 0.25]]},
    ],
    "param": [
        # A0 = diag(-1,-2), Bl = Br = e1, Q = I: v = 1 -> A = diag(-2,-2), X = diag(1/4, 1/4)
        {"A0": [[-1.0, 0.0], [0.0, -2.0]], "B": [[1.0], [0.0]], "Q": [[1.0, 0.0], [0.0, 1.0]],
         "E": [[1.0, 0.0], [0.0, 1.0]], "v": [1.0], "X": [[0.25, 0.0], [0.0, 0.25]], "trace": 0.5},
        # same problem, v = 3 -> A = diag(-4,-2), X = diag(1/8, 1/4)  (derived, same rule)
        {"A0": [[-1.0, 0.0], [0.0, -2.0]], "B": [[1.0], [0.0]], "Q": [[1.0, 0.0], [0.0, 1.0]],
         "E": [[1.0, 0.0], [0.0, 1.0]], "v": [3.0], "X": [[0.125, 0.0], [0.0, 0.25]], "trace": 0.375},
    ],
}
(out / "spec_examples.json").write_text(json.dumps(spec, indent=1))
print("wrote", out)

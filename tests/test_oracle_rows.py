"""hemm_step_rows is hemm_step restricted to a row panel (used for bounded CPU samples)."""
import numpy as np

import oracle
from chase_gen import make_matrix


def test_rows_equal_full_step():
    H = make_matrix("uniform", 90, "g2", seed=1).dense()
    rng = np.random.default_rng(0)
    X = rng.standard_normal((90, 5)) + 1j * rng.standard_normal((90, 5))
    Y = rng.standard_normal((90, 5)) + 1j * rng.standard_normal((90, 5))
    full = oracle.hemm_step(H, X, Y, 0.3, -0.7, 0.2)
    part = oracle.hemm_step_rows(H[30:55], 30, X, Y[30:55], 0.3, -0.7, 0.2)
    np.testing.assert_allclose(part, full[30:55], rtol=1e-14, atol=1e-15)

"""Input recipes shared by tools/gen_golden.py and the tests (no reference import)."""

from __future__ import annotations

import numpy as np


def rand_sym(n, seed):
    """conftest.py:11-14 generator (reference test contract)."""
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    return (G + G.T) / 2.0


def dense_suite():
    """(name, M) cases: reference KATs, the criterion-3 suite recipe
    (test_acceptance.py:79-97) and a few larger blocks."""
    cases = [("eye4", np.eye(4, dtype=complex)),
             ("swap2", np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex))]
    rng = np.random.default_rng(42)
    for t in range(200):
        n = int(rng.integers(2, 65))
        M = rand_sym(n, int(rng.integers(0, 2 ** 31)))
        if t % 2 == 0:
            for idx in rng.integers(0, n, size=min(3, n)):
                M[idx, idx] = 0.0
        cases.append((f"crit3_{t}", M))
    for n, seed in ((128, 7), (256, 8), (256, 9), (300, 10)):
        M = rand_sym(n, seed)
        M[np.diag_indices(n)] *= 0.1
        cases.append((f"big_{n}_{seed}", M))
    return cases

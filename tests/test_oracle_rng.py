"""Pins for the oracle-side counter-based generator (Philox4x32-10 known answers) -- CPU."""
import numpy as np

from oracle.rng import philox4x32_10, random_block


def _u(x):
    return int(x, 16) if isinstance(x, str) else int(x)


def test_philox_known_answers(golden):
    for case in golden("philox_kat.json")["cases"]:
        ctr = [np.array([_u(c)], dtype=np.uint32) for c in case["ctr"]]
        out = philox4x32_10(*ctr, _u(case["key"][0]), _u(case["key"][1]))
        assert [int(o[0]) for o in out] == [_u(x) for x in case["out"]]


def test_random_block_grid_invariant_and_range():
    full = random_block(2, 0, 100, 0, 7, 0)
    assert np.array_equal(random_block(2, 37, 20, 3, 4, 0), full[37:57, 3:7])
    assert np.all(np.abs(full.real) < 1) and np.all(np.abs(full.imag) < 1)
    assert abs(full.real.mean()) < 0.1 and abs(full.imag.mean()) < 0.1
    assert not np.array_equal(random_block(2, 0, 100, 0, 7, 1), full)

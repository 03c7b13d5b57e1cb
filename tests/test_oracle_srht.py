"""Oracle SRHT restatement pinned against the reference's own SRHT tests
(test_sketch.cpp:47-125, 252-285) -- CPU."""
import numpy as np
import pytest

from oracle import oracle as orc


def naive_hadamard(n):
    if n == 1:
        return np.ones((1, 1))
    h = naive_hadamard(n // 2)
    return np.block([[h, h], [h, -h]]) / np.sqrt(2.0)


def test_fast_transform_equals_recursive_definition():
    for n in (2, 4, 8, 16):
        x = np.random.default_rng(100 + n).standard_normal(n)
        assert np.max(np.abs(orc.hadamard_apply(x) - naive_hadamard(n) @ x)) < 1e-12
    t = orc.hadamard_apply(np.array([1.0, 0.0]))
    assert abs(t[0] - 1 / np.sqrt(2)) < 1e-15 and abs(t[1] - 1 / np.sqrt(2)) < 1e-15


def test_transform_involutive_norm_preserving():
    x = np.random.default_rng(7).standard_normal(1 << 16)
    hx = orc.hadamard_apply(x)
    assert abs(np.linalg.norm(hx) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(orc.hadamard_apply(hx) - x) <= 1e-12 * np.linalg.norm(x)
    with pytest.raises(orc.OracleError):
        orc.hadamard_apply(np.ones(3))


def test_sample_count_frozen_value():
    fv, c, capped = orc.srht_sample_count(1 << 20, 10, 0.5)
    assert abs(fv - 6633578.924774391) <= 1e-12 * 6633578.924774391
    assert capped and c == 1 << 20
    assert orc.srht_sample_count(1 << 20, 10, 0.9)[0] <= fv
    for args in ((5, 5, 0.5), (10, 0, 0.5), (100, 5, 0.0), (100, 5, 1.0)):
        with pytest.raises(orc.OracleError):
            orc.srht_sample_count(*args)


def test_srht_solve_accurate_deterministic_padded():
    rng = np.random.default_rng(41)
    a = rng.standard_normal((64, 2))
    b = a @ np.array([1.5, -0.75]) + 0.1 * rng.standard_normal(64)
    exact = np.linalg.lstsq(a, b, rcond=None)[0]
    good = sum(np.linalg.norm(orc.srht_solve(a, b, 64, 5000 + s)[0] - exact) / np.linalg.norm(exact) < 0.15
               for s in range(50))
    assert good >= 45
    a2 = rng.standard_normal((100, 3))
    b2 = a2 @ np.array([0.5, 2.0, -1.0]) + 0.1 * rng.standard_normal(100)
    ex2 = np.linalg.lstsq(a2, b2, rcond=None)[0]
    x = orc.srht_solve(a2, b2, 128, 9)[0]
    assert np.all(np.isfinite(x)) and np.linalg.norm(x - ex2) < 0.1 * np.linalg.norm(ex2)
    assert np.array_equal(orc.srht_solve(a2, b2, 64, 10)[0], orc.srht_solve(a2, b2, 64, 10)[0])
    with pytest.raises(orc.OracleError):
        orc.srht_solve(a2, b2, 2, 1)


def test_srht_fit_usage_errors():
    y = np.sin(np.arange(500) * 0.3) + 0.01 * np.arange(500)
    with pytest.raises(orc.OracleError):
        orc.srht_fit(y, 0, 100, 1)
    with pytest.raises(orc.OracleError):
        orc.srht_fit(y, 10, 5, 1)
    with pytest.raises(orc.OracleError):
        orc.srht_fit(y[:8], 10, 100, 1)

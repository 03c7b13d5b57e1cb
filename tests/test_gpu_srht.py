"""GPU SRHT path against the oracle restatement of
sketch.cpp:103-239 / bench.cpp:50-72 and the reference's SRHT tests
(test_sketch.cpp:47-100, 252-285).  Bars: transform 1e-12 against the
recursive definition; phi / PACF within 1e-9 of the oracle (the sampled rows
are bit-identical: same draws, same transform order); identical p*."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module")
def tf():
    import paper_2112_12994_b200 as t
    from paper_2112_12994_b200 import build
    build.build()
    return t


@pytest.fixture(scope="module")
def eng(tf):
    e = tf.Engine(0)
    yield e
    e.close()


def naive_hadamard(n):
    if n == 1:
        return np.ones((1, 1))
    h = naive_hadamard(n // 2)
    return np.block([[h, h], [h, -h]]) / np.sqrt(2.0)


def series(n, seed, q=6):
    from paper_2112_12994_b200 import gen
    return gen.simulate_roots(gen.ar_roots(q, 1.3, 3.0, seed), n, seed)


def relerr(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_transform_matches_definition_and_oracle(orc, tf, eng):
    for n in (2, 4, 8, 16):
        x = np.random.default_rng(100 + n).standard_normal(n)
        assert np.max(np.abs(tf.hadamard_apply(x, engine=eng) - naive_hadamard(n) @ x)) < 1e-12
    for m in (5, 11, 12, 17, 20):  # one contiguous pass, strided + contiguous, three passes
        x = np.random.default_rng(m).standard_normal(1 << m)
        assert relerr(tf.hadamard_apply(x, engine=eng), orc.hadamard_apply(x)) < 1e-13


def test_transform_involutive_and_rejects_bad_length(tf, eng):
    x = np.random.default_rng(7).standard_normal(1 << 16)
    hx = tf.hadamard_apply(x, engine=eng)
    assert abs(np.linalg.norm(hx) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
    assert np.linalg.norm(tf.hadamard_apply(hx, engine=eng) - x) <= 1e-12 * np.linalg.norm(x)
    with pytest.raises(tf.UsageError):
        tf.hadamard_apply(np.ones(3), engine=eng)


CASES = [  # n, p_bar, c  (N = bit_ceil(n - h): 1, 2 and 3 transform passes)
    (1500, 8, 300),
    (20000, 16, 2000),
    (300000, 10, 3000),
    (3000000, 4, 2000),
]


@pytest.mark.parametrize("n,p_bar,c", CASES)
def test_srht_fit_matches_oracle(orc, tf, eng, n, p_bar, c):
    y = series(n, seed=n % 97)
    ref = orc.srht_fit(y, p_bar, c, 4)
    fit = tf.srht_fit(tf.TimeSeries(y), p_bar, c, 4, engine=eng)
    assert relerr(fit.pacf.taus, ref.taus) < TOL
    for h in range(p_bar):
        assert relerr(fit.per_lag_coefficients[h], ref.coefs[h]) < TOL
    assert fit.p_star == ref.p_star
    assert abs(fit.pacf.bound - 1.96 / np.sqrt(c)) < 1e-15


def test_srht_run_fit_deterministic_and_errors(tf, eng):
    y = series(5000, 3)
    a = tf.run_fit(tf.TimeSeries(y), "srht", 8, 300, 4, engine=eng)
    b = tf.run_fit(tf.TimeSeries(y), "srht", 8, 300, 4, engine=eng)
    c = tf.run_fit(tf.TimeSeries(y), "srht", 8, 300, 5, engine=eng)
    assert a.method == "srht" and a.pacf.taus == b.pacf.taus and a.pacf.taus != c.pacf.taus
    with pytest.raises(tf.UsageError):
        tf.srht_fit(tf.TimeSeries(y), 0, 300, 1, engine=eng)
    with pytest.raises(tf.UsageError):
        tf.srht_fit(tf.TimeSeries(y), 10, 5, 1, engine=eng)
    with pytest.raises(tf.DataError):
        tf.srht_fit(tf.TimeSeries(y[:8]), 10, 100, 1, engine=eng)

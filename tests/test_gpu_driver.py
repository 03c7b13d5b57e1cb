"""LsarDriver step API on the GPU (lsar.hpp:65-84, lsar.cpp:55-98) through
tf_lsar_step: GPU port of test_lsar.cpp:130-158 ("driver advances the state
with constant row count"), the reference's error cases, and the step API
against the fused sweep (stepping with the device-resident state is the same
launch sequence as tf_lsar_sweep: bit-identical) and against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


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


def test_driver_advances_with_constant_row_count(orc, tf, eng):
    # test_lsar.cpp:130-158
    y = orc.simulate_ar(orc.random_stationary_ar(2, 221), 800, 222)
    drv = tf.LsarDriver(tf.TimeSeries(y), 10, 120, 9, engine=eng)
    assert drv.row_count() == 790
    s1 = drv.first_lag()
    assert s1.p == 1 and s1.m == 791
    assert s1.scores.size == 790 and s1.residuals.size == 790 and s1.coefficients.size == 1
    assert np.max(np.abs(s1.scores - orc.init_leverage_p1(y[:790]))) < 1e-15
    s2 = drv.advance(s1)
    assert s2.p == 2 and s2.m == 792 and s2.scores.size == 790 and s2.coefficients.size == 2
    assert abs(s2.scores.sum() - 2.0) < 1e-12
    assert (s2.scores - s1.scores).min() >= -1e-15
    # replays are deterministic
    r1 = drv.first_lag()
    assert np.array_equal(r1.coefficients, s1.coefficients)
    r2 = drv.advance(r1)
    assert np.array_equal(r2.coefficients, s2.coefficients)


def test_driver_errors(tf, eng):
    y = np.sin(np.arange(50) * 0.3) + 0.01 * np.arange(50)
    s = tf.TimeSeries(y)
    with pytest.raises(tf.UsageError):
        tf.LsarDriver(s, 10, 5, 1, engine=eng)      # c below the maximum lag
    with pytest.raises(tf.DataError):
        tf.LsarDriver(s, 49, 100, 1, engine=eng)    # series too short
    with pytest.raises(tf.UsageError):
        tf.LsarDriver(s, 0, 100, 1, engine=eng)
    drv = tf.LsarDriver(s, 2, 20, 1, engine=eng)
    st = drv.advance(drv.first_lag())
    with pytest.raises(tf.UsageError, match="cannot advance past maximum lag"):
        drv.advance(st)
    geo = tf.TimeSeries(0.5 ** np.arange(60))       # test_lsar.cpp:160-169: zero residual
    with pytest.raises(tf.NumericalError):
        d = tf.LsarDriver(geo, 3, 20, 1, engine=eng)
        d.advance(d.advance(d.first_lag()))


def test_driver_steps_equal_the_fused_sweep(tf, eng):
    from paper_2112_12994_b200 import gen
    y = gen.simulate_roots(gen.ar_roots(8, 1.2, 3.0, 5), 60000, 5)
    s = tf.TimeSeries(y)
    p_bar, c, seed = 20, 3000, 33
    fit = tf.lsar_fit(s, p_bar, c, seed, engine=eng)
    drv = tf.LsarDriver(s, p_bar, c, seed, engine=eng)
    st = drv.first_lag()
    coefs = [st.coefficients]
    while st.p < p_bar:
        st = drv.advance(st)  # the state the previous call returned: device-resident continuation
        coefs.append(st.coefficients)
    for p in range(p_bar):
        assert np.array_equal(coefs[p], fit.per_lag_coefficients[p])


def test_driver_host_state_round_trip(tf, eng):
    # advancing a copy of a state (host vectors uploaded) gives the same lag as
    # continuing from the resident one
    from paper_2112_12994_b200 import gen
    y = gen.simulate_roots(gen.ar_roots(4, 1.3, 3.0, 8), 30000, 8)
    s = tf.TimeSeries(y)
    drv = tf.LsarDriver(s, 6, 1500, 4, engine=eng)
    a = drv.advance(drv.first_lag())
    copy = tf.LeverageState(p=a.p, m=a.m, scores=a.scores.copy(), residuals=a.residuals.copy(),
                            coefficients=a.coefficients.copy())
    b_res = drv.advance(a)
    b_host = drv.advance(copy)
    assert b_host.p == b_res.p == 3
    # the uploaded state re-derives the CDF partials (k_partials): the same
    # distribution up to summation order -> the same draws in practice
    assert np.max(np.abs(b_host.coefficients - b_res.coefficients)) <= 1e-9 * np.max(np.abs(b_res.coefficients))
    assert np.max(np.abs(b_host.scores - b_res.scores)) <= 1e-15 * np.max(b_res.scores)

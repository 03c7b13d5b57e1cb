"""GPU exact per-lag OLS (bench.cpp:27-48) against the
oracle's restatement (Householder CPQR per lag on the full series)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def relerr(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("n,q,p_bar", [(20000, 6, 12), (60000, 20, 40), (200000, 20, 60)])
def test_exact_fit_matches_oracle(orc, n, q, p_bar):
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen
    y = gen.simulate_roots(gen.ar_roots(q, 1.2, 3.0, n + q), n, n + q)
    ref = orc.exact_fit(y, p_bar)
    eng = tf.Engine(0)
    fit = tf.exact_fit(tf.TimeSeries(y), p_bar, engine=eng)
    assert relerr(fit.pacf.taus, ref.taus) < 1e-9
    for h in range(p_bar):
        assert relerr(fit.per_lag_coefficients[h], ref.coefs[h]) < 1e-9
    assert fit.p_star == ref.p_star
    assert abs(fit.pacf.bound - 1.96 / np.sqrt(n - p_bar)) < 1e-15
    rep = tf.run_fit(tf.TimeSeries(y), "exact", p_bar, 0, 1, engine=eng)
    assert rep.p_star == ref.p_star
    eng.close()

"""Batched LSAR sweeps (tf_lsar_sweep_batch): many independent fits per launch.

Each fit of a batch must equal lsar_fit of its own series and seed
(lsar.cpp:100-124): in deterministic-index mode phi / PACF within rel 1e-9 of
the oracle with identical p*; in RNG mode the same draws as the single-series
path (so the same taus to 1e-9) except where a draw lands within rounding of a
CDF boundary.  A fit whose sampled system breaks down is re-run through the
single-series path, so it equals lsar_fit exactly.
"""
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


def series(n, q, seed, lo=1.1, hi=3.0):
    from paper_2112_12994_b200 import gen
    return gen.simulate_roots(gen.ar_roots(q, lo, hi, seed), n, seed)


def relerr(a, b):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("n,p_bar,c", [(6000, 20, 600), (20000, 50, 2000), (3000, 63, 300), (2100, 5, 40)])
def test_batch_fixed_index_parity(orc, tf, eng, n, p_bar, c):
    qs = [1, 3, 7, 10, 2]
    ys = [series(n, q, 100 + k) for k, q in enumerate(qs)]
    seeds = [11 + k for k in range(len(ys))]
    refs = [orc.lsar_fit(y, p_bar, c, s) for y, s in zip(ys, seeds)]
    fi = np.stack([r.idx for r in refs])
    fw = np.stack([r.w for r in refs])
    fits = tf.lsar_fit_batch(ys, p_bar, c, seeds, engine=eng, fixed_idx=fi, fixed_w=fw)
    for f, r in zip(fits, refs):
        assert relerr(f.pacf.taus, r.taus) < TOL
        for p in range(p_bar):
            assert relerr(f.per_lag_coefficients[p], r.coefs[p]) < TOL
        assert f.p_star == r.p_star


def test_batch_rng_mode_matches_single_path(orc, tf, eng):
    n, p_bar, c = 30000, 30, 1500
    ys = [series(n, q, 300 + q) for q in (1, 4, 9, 6, 2, 10)]
    seeds = [7000 + k for k in range(len(ys))]
    fits = tf.lsar_fit_batch(ys, p_bar, c, seeds, engine=eng)
    close = 0
    for y, s, f in zip(ys, seeds, fits):
        g = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, s, engine=eng)
        if relerr(f.pacf.taus, g.pacf.taus) < TOL:
            close += 1
            assert f.p_star == g.p_star
        r = orc.lsar_fit(y, p_bar, c, s)
        # lag 1 samples from closed-form scores: the same draws as the oracle
        assert abs(f.pacf.taus[0] - r.taus[0]) <= TOL * abs(r.taus[0])
    assert close >= len(ys) - 1


def test_batch_shared_series_equals_copies(tf, eng):
    y = series(12000, 5, 9)
    seeds = [1, 2, 3, 4]
    a = tf.lsar_fit_batch(tf.TimeSeries(y), 12, 800, seeds, engine=eng)
    b = tf.lsar_fit_batch([y] * 4, 12, 800, seeds, engine=eng)
    for f, g in zip(a, b):
        assert f.pacf.taus == g.pacf.taus
    assert a[0].pacf.taus != a[1].pacf.taus  # seeds matter
    c = tf.lsar_fit_batch(tf.TimeSeries(y), 12, 800, seeds, engine=eng)  # deterministic
    assert [f.pacf.taus for f in a] == [f.pacf.taus for f in c]


def test_batch_errors_per_fit(tf, eng):
    geo = 0.5 ** np.arange(200)  # zero residual at lag 2 (test_lsar.cpp:160-169)
    y = series(200, 2, 5)
    fits = tf.lsar_fit_batch([y, geo, y], 3, 20, [1, 1, 2], engine=eng, errors="return")
    assert isinstance(fits[1], tf.NumericalError)
    assert not isinstance(fits[0], Exception) and not isinstance(fits[2], Exception)
    g = tf.lsar_fit(tf.TimeSeries(y), 3, 20, 1, engine=eng)
    assert relerr(fits[0].pacf.taus, g.pacf.taus) < 1e-6
    with pytest.raises(tf.NumericalError):
        tf.lsar_fit_batch([y, geo], 3, 20, [1, 1], engine=eng)
    with pytest.raises(tf.UsageError):
        tf.lsar_fit_batch([y, y], 64, 200, [1, 2], engine=eng)  # p_bar above the batched limit
    with pytest.raises(tf.UsageError):
        tf.lsar_fit_batch([y, y], 10, 5, [1, 2], engine=eng)  # c < p_bar
    with pytest.raises(tf.DataError):
        tf.lsar_fit_batch([y[:20], y[:20]], 19, 40, [1, 2], engine=eng)
    with pytest.raises(tf.UsageError):
        tf.lsar_fit_batch([y, y[:100]], 3, 20, [1, 2], engine=eng)  # ragged batch


def test_batch_rank_deficient_fit_falls_back(tf, eng):
    # c = p_bar: the lag-p_bar system has more columns than rows -> the
    # single-series path's minimum-norm answer, bit-identical to lsar_fit
    ys = [series(4000, 3, 40 + k) for k in range(3)]
    fits = tf.lsar_fit_batch(ys, 10, 10, [5, 6, 7], engine=eng)
    for y, s, f in zip(ys, [5, 6, 7], fits):
        g = tf.lsar_fit(tf.TimeSeries(y), 10, 10, s, engine=eng)
        assert f.pacf.taus == g.pacf.taus


def test_upload_rejects_non_finite_through_the_abi(tf, eng):
    # series.cpp:23-32 through tf_upload_series itself (the host mirror's
    # TimeSeries check bypassed): DataError with the first bad position, and
    # no series stays resident
    import ctypes as C
    from paper_2112_12994_b200 import _abi
    y = np.arange(10.0)
    y[7] = np.inf
    y[8] = np.nan
    st = _abi.lib().tf_upload_series(eng._ctx, _abi.ptr(y), y.size)
    assert st == _abi.TF_DATA
    assert "position 7" in _abi.lib().tf_last_error(eng._ctx).decode()
    taus = np.zeros(2)
    st = _abi.lib().tf_lsar_sweep(eng._ctx, 2, 4, C.c_uint64(1), None, _abi.ptr(taus), None, None, None)
    assert st == _abi.TF_USAGE  # "no series uploaded"
    eng._series_id = None

"""GPU parity of the Repeated-Halving sweep against the oracle (through the C ABI).

Bars: halving index sets bit-exact (integer work, same counter RNG); in
deterministic-index mode (levels, upward samples and per-lag samples taken
from the oracle) final leverage scores, phi and PACF within rel 1e-9 and the
same p*; RNG mode: identical upward / per-lag draws in practice.
Reference: repeated_halving.cpp:126-232, test_repeated_halving.cpp.
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


def c1_like(n, seed=5, q=20, lo=1.2, hi=3.0):
    from paper_2112_12994_b200 import gen
    roots = gen.ar_roots(q, lo, hi, seed)
    return gen.simulate_roots(roots, n, seed)


def relerr(a, b):
    a = np.asarray(a, float); b = np.asarray(b, float)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


CASES = [  # n, q, p_bar, c
    (30000, 5, 8, 200),
    (60000, 20, 30, 1500),
    (40000, 10, 70, 800),
]


@pytest.mark.parametrize("n,q,p_bar,c", CASES)
def test_rh_levels_bit_exact(orc, tf, eng, n, q, p_bar, c):
    y = c1_like(n, seed=n + q, q=q)
    ref = orc.rh_fit(y, p_bar, c, 31, want_levels=True)
    fit = tf.rh_fit(tf.TimeSeries(y), p_bar, c, None, 31, engine=eng, want_diag=True)
    d = fit.diag
    assert d["depth"] == ref.depth and ref.depth >= 2
    assert list(d["level_sizes"]) == list(ref.level_sizes)
    for lv_gpu, lv_ref in zip(d["levels"], ref.levels):
        assert np.array_equal(lv_gpu, lv_ref)


@pytest.mark.parametrize("n,q,p_bar,c", CASES)
def test_rh_fixed_index_parity(orc, tf, eng, n, q, p_bar, c):
    y = c1_like(n, seed=n + q + 1, q=q)
    ref = orc.rh_fit(y, p_bar, c, 9, want_levels=True)
    flat = np.concatenate(ref.levels) if ref.levels else np.zeros(0, np.int64)
    fixed = dict(idx=ref.idx, w=ref.w, levels=flat, up_idx=ref.up_idx, up_w=ref.up_w)
    fit = tf.rh_fit(tf.TimeSeries(y), p_bar, c, None, 9, engine=eng, fixed=fixed, want_diag=True)
    d = fit.diag
    assert np.array_equal(d["idx"], ref.idx)
    assert relerr(d["scores"], ref.scores) < TOL
    assert relerr(fit.pacf.taus, ref.taus) < TOL
    for p in range(p_bar):
        assert relerr(fit.per_lag_coefficients[p], ref.coefs[p]) < TOL
    assert fit.p_star == ref.p_star


def test_rh_rng_mode_matches_oracle_draws(orc, tf, eng):
    n, q, p_bar, c = 60000, 20, 30, 1500
    y = c1_like(n, seed=3, q=q)
    ref = orc.rh_fit(y, p_bar, c, 5, want_levels=True)
    fit = tf.rh_fit(tf.TimeSeries(y), p_bar, c, None, 5, engine=eng, want_diag=True)
    d = fit.diag
    # upward samples: same counter draws on scores equal to ~1e-15
    agree_up = np.mean(d["up_idx"] == ref.up_idx)
    assert agree_up >= 0.999
    assert relerr(d["scores"], ref.scores) < 1e-8
    agree = np.mean(d["idx"] == ref.idx)
    assert agree >= 0.999
    assert fit.p_star == ref.p_star
    assert relerr(fit.pacf.taus, ref.taus) < 1e-6


def test_rh_depth_zero_and_explicit_config(orc, tf, eng):
    # m <= base threshold: no halving, final scores against all rows
    y = c1_like(3000, seed=11, q=4)
    p_bar, c = 6, 400
    cfg = tf.RHConfig(base_threshold=5000, sample_count=400, gaussian_rows=20, seed=77)
    ocfg = orc.rh_defaults(y.size - p_bar, p_bar + 1, c, 77)
    ocfg.base_threshold, ocfg.sample_count, ocfg.gaussian_rows, ocfg.seed = 5000, 400, 20, 77
    ref = orc.rh_fit(y, p_bar, c, 2, cfg=ocfg)
    fit = tf.rh_fit(tf.TimeSeries(y), p_bar, c, cfg, 2, engine=eng, fixed=dict(idx=ref.idx, w=ref.w),
                    want_diag=True)
    assert fit.diag["depth"] == 0 == ref.depth
    assert relerr(fit.diag["scores"], ref.scores) < TOL
    assert relerr(fit.pacf.taus, ref.taus) < TOL
    # scores of the exact leverage against all rows sum to k (trace of the hat matrix)
    assert abs(fit.diag["scores"].sum() - (p_bar + 1)) < 1e-8


def test_rh_deterministic(tf, eng):
    y = c1_like(20000, seed=2, q=6)
    a = tf.rh_fit(tf.TimeSeries(y), 10, 500, None, 4, engine=eng)
    b = tf.rh_fit(tf.TimeSeries(y), 10, 500, None, 4, engine=eng)
    c = tf.rh_fit(tf.TimeSeries(y), 10, 500, None, 5, engine=eng)
    assert a.pacf.taus == b.pacf.taus
    assert a.pacf.taus != c.pacf.taus


def test_rh_errors(tf, eng):
    y = c1_like(2000, seed=1, q=3)
    with pytest.raises(tf.UsageError):
        tf.rh_fit(tf.TimeSeries(y), 10, 5, None, 1, engine=eng)  # c < p_bar
    with pytest.raises(tf.UsageError):
        tf.rh_fit(tf.TimeSeries(y), 4, 100, tf.RHConfig(50, 100, 8, 1), 1, engine=eng)  # base < sc
    with pytest.raises(tf.UsageError):
        tf.rh_fit(tf.TimeSeries(y), 4, 100, tf.RHConfig(200, 100, 0, 1), 1, engine=eng)  # g < 1
    with pytest.raises(tf.DataError):
        tf.rh_fit(tf.TimeSeries(y[:5]), 4, 100, None, 1, engine=eng)
    with pytest.raises(tf.NumericalError):  # approximation rows < k
        tf.rh_fit(tf.TimeSeries(y), 20, 25, tf.RHConfig(30, 10, 8, 1), 1, engine=eng)


def test_fit_many_matches_sequential(tf, eng):
    # concurrent contexts give exactly the sequential results (same kernels, same seeds)
    ys = [c1_like(8000 + 500 * k, seed=40 + k, q=4) for k in range(6)]
    seeds = [3 + k for k in range(6)]
    many = tf.fit_many(ys, "lsar", 10, 300, seeds, workers=3)
    for y, s, f in zip(ys, seeds, many):
        ref = tf.lsar_fit(tf.TimeSeries(y), 10, 300, s, engine=eng)
        assert f.pacf.taus == ref.pacf.taus and f.p_star == ref.p_star
    rh = tf.fit_many(ys[:3], "rh", 8, 300, seeds[:3], workers=3)
    for y, s, f in zip(ys[:3], seeds[:3], rh):
        ref = tf.rh_fit(tf.TimeSeries(y), 8, 300, None, s, engine=eng)
        assert f.pacf.taus == ref.pacf.taus

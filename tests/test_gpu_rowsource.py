"""Repeated Halving over a general RowSource on the GPU
(repeated_halving.hpp:17-23, 76-91): GPU ports of test_rh.cpp:61-141 and
oracle parity of generalized_leverage (sketched and unsketched) and of the
halving + upward pass on dense matrices."""
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


def rmat(rows, cols, seed):
    return np.random.default_rng(seed).standard_normal((rows, cols))


def test_generalized_leverage_against_itself_is_exact(orc, tf, eng):
    # test_rh.cpp:61-76
    d = np.random.default_rng(11)
    for trial in range(10):
        cols = 1 + int(d.integers(0, 15))
        rows = cols + 1 + int(d.integers(0, 285))
        a = rmat(rows, cols, 100 + trial)
        gen = tf.generalized_leverage(a, a, None, engine=eng)
        assert np.max(np.abs(gen - orc.exact_leverage(a))) < 1e-10
    eye = np.eye(6)
    assert np.allclose(tf.generalized_leverage(eye, eye, None, engine=eng), 1.0, rtol=1e-14, atol=0)


def test_generalized_leverage_validates(tf, eng):
    # test_rh.cpp:78-89
    c = rmat(20, 3, 21)
    with pytest.raises(tf.UsageError):
        tf.generalized_leverage(c, rmat(20, 4, 22), None, engine=eng)
    dup = np.empty((20, 3))
    dup[:, 0] = rmat(20, 1, 23)[:, 0]
    dup[:, 1] = dup[:, 0]
    dup[:, 2] = rmat(20, 1, 24)[:, 0]
    with pytest.raises(tf.NumericalError, match="rank deficient"):
        tf.generalized_leverage(c, dup, None, engine=eng)
    with pytest.raises(tf.NumericalError, match="too few rows"):
        tf.generalized_leverage(c, rmat(2, 3, 25), None, engine=eng)


def test_sketched_generalized_leverage(orc, tf, eng):
    # test_rh.cpp:91-103 (concentration) and the oracle's sketch, same normals
    a = rmat(512, 8, 31)
    exact = tf.generalized_leverage(a, a, None, engine=eng)
    approx = tf.generalized_leverage(a, a, tf.GaussianSketch(64, 32), engine=eng)
    ratio = approx / exact
    assert np.sum((ratio >= 1 / 3) & (ratio <= 3)) >= 487
    ref = orc.generalized_leverage(a, a, 64, 32)
    assert np.max(np.abs(approx - ref) / np.abs(ref)) < 1e-9


def test_halving_identity_at_base(tf, eng):
    # test_rh.cpp:105-116
    a = rmat(100, 5, 41)
    cfg = tf.RHConfig(base_threshold=128, sample_count=64, gaussian_rows=16, seed=7)
    ap = tf.repeated_halving(tf.DenseRowSource(a), cfg, engine=eng)
    assert ap.levels == 0 and np.array_equal(ap.rows, a)


def test_halved_approximation_preserves_rank_and_sandwiches(tf, eng):
    # test_rh.cpp:118-141
    x = rmat(512, 6, 51)
    cfg = tf.RHConfig(base_threshold=128, sample_count=128, gaussian_rows=48, seed=3)
    ap = tf.repeated_halving(tf.DenseRowSource(x), cfg, engine=eng)
    assert ap.levels == 2 and ap.rows.shape == (128, 6)
    assert np.linalg.matrix_rank(ap.rows) == 6
    inside = 0
    for t in range(50):
        v = rmat(6, 1, 600 + t)[:, 0]
        v /= np.linalg.norm(v)
        full, sk = np.sum((x @ v) ** 2), np.sum((ap.rows @ v) ** 2)
        inside += 0.4 * full <= sk <= 2.5 * full
    assert inside >= 45


def test_repeated_halving_matches_oracle_on_augmented_rows(orc, tf, eng):
    # the same halving draws and upward samples as the oracle's rh_fit on the
    # augmented lag-p_bar system: the approximation rows agree to ~1e-12
    y = orc.simulate_ar(orc.random_stationary_ar(3, 71), 2052, 72)
    p_bar = 4
    cfg = orc.RhCfg(600, 200, 24, 5)
    ref = orc.rh_fit(y, p_bar, 200, 9, cfg=cfg)
    ap = tf.repeated_halving(tf.AugmentedRowSource(tf.TimeSeries(y), p_bar),
                             tf.RHConfig(base_threshold=600, sample_count=200, gaussian_rows=24, seed=5), engine=eng)
    assert ap.levels == ref.depth == 2
    assert np.max(np.abs(ap.rows - ref.approx)) <= 1e-12 * np.max(np.abs(ref.approx))


def test_score_pass_at_base_is_exact_leverage(orc, tf, eng):
    # test_rh.cpp:143-155: at or below the base the scores are exact leverage of [T, b]
    y = orc.simulate_ar(orc.random_stationary_ar(2, 61), 60, 62)
    s = tf.TimeSeries(y)
    cfg = tf.RHConfig(base_threshold=64, sample_count=32, gaussian_rows=16, seed=5)
    sc = tf.rh_leverage_scores(s, 4, cfg, engine=eng)
    aug = tf.AugmentedRowSource(s, 4).gather(np.arange(56))
    assert np.max(np.abs(sc - orc.exact_leverage(aug))) < 1e-10

"""GPU parity of the FFT pass (k_fft.cuh: overlap-save FFT FIR + leverage
update + CDF partials) -- the pass the sweeps run for the long lags.

TF_PASS=fft forces it at every lag q >= 1 (TF_PASS=dmma: the direct
tensor-core FIR only); the variable is read when an Engine is created.

Bars (BASELINE.json north_star): sampled indices bit-exact in
deterministic-index mode; scores, residuals, phi, PACF within rel 1e-9 of the
oracle (the reference's tap-order FIR); identical p*; RNG-mode draws identical
up to a neighbouring-row rounding flip.  Shapes cover the superblock edges
(w below one 3072-row block, exactly one 6144-row superblock, one row past
it, many superblocks) and the largest lag a sweep takes (q = 640, the solve's
limit; the blocks hold q <= D = 1024), where the oracle's own solve is too
slow: there the FFT
sweep is compared with the direct-FIR sweep on identical fixed draws and
weights (identical sampled systems, so phi is bit-identical and only the
FIR's rounding differs).
"""
import numpy as np
import pytest

from test_gpu_lsar import c1_like, check_flip, relerr

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def tf():
    import paper_2112_12994_b200 as t
    from paper_2112_12994_b200 import build
    build.build()
    return t


def engine(tf, monkeypatch, mode):
    monkeypatch.setenv("TF_PASS", mode)
    e = tf.Engine(0)
    monkeypatch.delenv("TF_PASS")
    return e


@pytest.mark.parametrize("n,q,p_bar,c", [(1000, 3, 3, 200), (6000, 4, 5, 300), (6149, 4, 5, 300),
                                         (6150, 4, 5, 300), (20000, 12, 40, 600), (45000, 20, 150, 1200)])
def test_fft_pass_fixed_index_parity(orc, tf, monkeypatch, n, q, p_bar, c):
    y = c1_like(n, seed=q + n, q=q)
    ref = orc.lsar_fit(y, p_bar, c, 91)
    eng = engine(tf, monkeypatch, "fft")
    try:
        fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, 91, engine=eng, fixed_idx=ref.idx, fixed_w=ref.w,
                          want_diag=True)
    finally:
        eng.close()
    d = fit.diag
    assert np.array_equal(d["idx"], ref.idx)
    assert relerr(fit.pacf.taus, ref.taus) < TOL
    for p in range(p_bar):
        assert relerr(fit.per_lag_coefficients[p], ref.coefs[p]) < TOL
    assert relerr(d["scores"], ref.scores) < TOL
    assert relerr(d["resid"], ref.resid) < TOL
    assert relerr(d["rnorm2"], ref.rnorm2) < TOL
    assert relerr(d["ssum"], ref.ssum) < TOL
    assert fit.p_star == ref.p_star
    assert abs(d["scores"].sum() - p_bar) < 1e-8


def test_fft_auto_mode_parity(orc, tf, monkeypatch):
    # default (auto) mode: direct FIR below the crossover lag, FFT from it on
    # (TF_FFT_MINQ lowered so a small fit crosses it)
    y = c1_like(30000, seed=8, q=10)
    p_bar, c = 30, 800
    ref = orc.lsar_fit(y, p_bar, c, 5)
    monkeypatch.setenv("TF_FFT_MINQ", "11")
    eng = tf.Engine(0)
    monkeypatch.delenv("TF_FFT_MINQ")
    try:
        fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, 5, engine=eng, fixed_idx=ref.idx, fixed_w=ref.w,
                          want_diag=True)
    finally:
        eng.close()
    assert relerr(fit.pacf.taus, ref.taus) < TOL
    assert relerr(fit.diag["scores"], ref.scores) < TOL
    assert relerr(fit.diag["resid"], ref.resid) < TOL
    assert relerr(fit.diag["rnorm2"], ref.rnorm2) < TOL
    assert fit.p_star == ref.p_star


def test_fft_rng_mode_matches_oracle_draws(orc, tf, monkeypatch):
    eng = engine(tf, monkeypatch, "fft")
    try:
        for n, q, p_bar, c, seed in [(30000, 20, 25, 2500, 4242), (12000, 4, 6, 900, 99)]:
            y = c1_like(n, seed=q + 3, q=q)
            ref = orc.lsar_fit(y, p_bar, c, seed)
            fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, seed, engine=eng, want_diag=True)
            flip = check_flip(fit.diag["idx"], ref.idx, c)
            upto = p_bar if flip is None else flip
            for p in range(upto):
                assert np.array_equal(fit.diag["idx"][p], ref.idx[p])
                assert relerr(fit.per_lag_coefficients[p], ref.coefs[p]) < TOL
            if flip is None:
                assert relerr(fit.pacf.taus, ref.taus) < TOL
                assert fit.p_star == ref.p_star
    finally:
        eng.close()


def test_fft_longest_lag_vs_direct(tf, monkeypatch):
    """q up to 640, the largest p_bar the rank-revealing solve takes (the
    4096-point blocks hold filters up to q = D = 1024)."""
    p_bar = 640
    n, c = 26000, 1100
    y = c1_like(n, seed=3, q=30)
    rng = np.random.default_rng(11)
    w = n - p_bar
    idx = rng.integers(0, w, size=(p_bar, c))
    wt = rng.uniform(0.5, 2.0, size=(p_bar, c))
    out = {}
    for mode in ("fft", "dmma"):
        eng = engine(tf, monkeypatch, mode)
        try:
            out[mode] = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, 1, engine=eng, fixed_idx=idx, fixed_w=wt,
                                    want_diag=True)
        finally:
            eng.close()
    f, g = out["fft"], out["dmma"]
    # identical sampled systems -> identical phi; the window residuals differ by FIR rounding only
    assert np.array_equal(np.array(f.pacf.taus), np.array(g.pacf.taus))
    assert relerr(f.diag["rnorm2"], g.diag["rnorm2"]) < TOL
    assert relerr(f.diag["ssum"], g.diag["ssum"]) < TOL
    assert relerr(f.diag["scores"], g.diag["scores"]) < TOL
    phi = np.asarray(f.per_lag_coefficients[-1])
    noise = 64 * np.finfo(float).eps * (1.0 + np.abs(phi).sum()) * np.max(np.abs(y))
    assert np.max(np.abs(f.diag["resid"] - g.diag["resid"])) < noise


def _exact_resid(seg, phi):
    """r(i) = -y[q + i] + sum_j phi[j] y[q - 1 - j + i] in long double (the
    reference for both fp64 FIRs)"""
    q = phi.size
    yl = seg.astype(np.longdouble)
    rows = seg.size - q
    r = -yl[q:q + rows].copy()
    for j in range(q):
        r += np.longdouble(phi[j]) * yl[q - 1 - j:q - 1 - j + rows]
    return r


def test_fft_spectra_accuracy_c2(orc, tf, monkeypatch):
    """BASELINE C2 (AR(50), n = 1e7, p_bar = 200): the FFT pass's residuals at
    the last lag against long-double residuals of the same phi.  The spectra
    are double-double, rounded once (k_fft_series_dd / k_fft_taps_dd), so the
    FFT residuals are at least as accurate as the oracle's direct fp64 tap
    loop (a plain fp64 FFT was at 1.6e-9 of max|r| here; the direct FIR is at
    4.9e-10)."""
    from paper_2112_12994_b200 import gen
    y, _, p_bar, _ = gen.make_config_series("C2")
    eng = engine(tf, monkeypatch, "fft")
    try:
        fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, 10_000, 99, engine=eng, want_diag=True)
    finally:
        eng.close()
    phi = np.asarray(fit.per_lag_coefficients[-1], float)
    w = y.size - p_bar
    worst_fft = worst_dir = 0.0
    for i0 in (0, w // 3, w - 6000):
        seg = y[i0:i0 + 6000 + p_bar]
        ex = _exact_resid(seg, phi)
        scale = float(np.max(np.abs(ex)))
        worst_fft = max(worst_fft, float(np.max(np.abs(fit.diag["resid"][i0:i0 + 6000] - ex))) / scale)
        worst_dir = max(worst_dir, float(np.max(np.abs(orc.residuals(seg, seg.size, p_bar, phi) - ex))) / scale)
    assert worst_fft < 1e-9, worst_fft
    assert worst_fft <= 1.5 * worst_dir, (worst_fft, worst_dir)


def test_fft_first_lag_abi(tf, monkeypatch):
    """tf_fft_first_lag: the auto crossover, the forced modes, p_bar past the
    4096-point blocks' filter length (direct FIR only)"""
    e = tf.Engine(0)
    try:
        assert e.fft_first_lag(500) == 64
        assert e.fft_first_lag(96) == 64
        assert e.fft_first_lag(95) == 96  # too few lags past the crossover to pay for the series spectra
        assert e.fft_first_lag(50) == 51  # below the crossover: no FFT lag
        assert e.fft_first_lag(2000) == 2001  # q > D = 1024: direct FIR only
    finally:
        e.close()
    for mode, want in (("fft", 1), ("dmma", 501)):
        e = engine(tf, monkeypatch, mode)
        try:
            assert e.fft_first_lag(500) == want
        finally:
            e.close()


def test_fft_split_score_update_equals_fused(tf, monkeypatch):
    """The score update of an FFT lag on its own stream beside the solve
    (k_fft_fold, TF_FFT_SPLIT=1, the default) against the update fused into the
    pass (TF_FFT_SPLIT=0): the same device code, so draws, fits, scores and
    residuals are bit-identical -- in RNG mode, three sweeps each (eager, the
    graph's capture, its replay).  One fold per lag (TF_FFT_SLOTS=1) applies the
    same fma sequence per row, but its chunk sums are reduced from the rows
    instead of advanced by the chunk recurrence, so the CDF totals -- and
    through the weights the fit, the residuals and the scores -- agree to
    rounding (1e-11), not bit for bit."""
    y = c1_like(60000, seed=17, q=9)
    p_bar, c = 24, 900
    out = {}
    for name, env in (("split", {"TF_FFT_SPLIT": "1"}), ("fused", {"TF_FFT_SPLIT": "0"}),
                      ("perlag", {"TF_FFT_SPLIT": "0", "TF_FFT_SLOTS": "1"})):
        monkeypatch.setenv("TF_PASS", "fft")
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        eng = tf.Engine(0)
        for k in ("TF_PASS", *env):
            monkeypatch.delenv(k)
        try:
            fits = [tf.lsar_fit(tf.TimeSeries(y), p_bar, c, 33, engine=eng, want_diag=True) for _ in range(3)]
        finally:
            eng.close()
        for f in fits[1:]:
            assert np.array_equal(f.diag["idx"], fits[0].diag["idx"])
            assert np.array_equal(np.array(f.pacf.taus), np.array(fits[0].pacf.taus))
            assert np.array_equal(f.diag["scores"], fits[0].diag["scores"])
        out[name] = fits[-1]
    a, b, k1 = out["split"], out["fused"], out["perlag"]
    assert np.array_equal(a.diag["idx"], b.diag["idx"])
    assert np.array_equal(np.array(a.pacf.taus), np.array(b.pacf.taus))
    assert np.array_equal(a.diag["scores"], b.diag["scores"])
    assert np.array_equal(a.diag["resid"], b.diag["resid"])
    assert np.array_equal(a.diag["ssum"], b.diag["ssum"])
    assert a.p_star == b.p_star == k1.p_star
    if np.array_equal(a.diag["idx"], k1.diag["idx"]):
        assert relerr(a.pacf.taus, k1.pacf.taus) < 1e-11
        assert relerr(a.diag["scores"], k1.diag["scores"]) < 1e-11
        assert relerr(a.diag["ssum"], k1.diag["ssum"]) < 1e-12
    else:
        check_flip(a.diag["idx"], k1.diag["idx"], c)

"""Pin the CPU oracle (oracle/) before trusting it.

1. Bit-exact against known answers produced by the reference's OWN rng.hpp
   (tests/golden/rng_kat.json, made by oracle/make_golden.py).
2. The reference's unit-test known answers and tolerance properties for this
   path (proj/tests/test_{toeplitz,sketch,lsar,rh}.cpp), restated against
   the oracle.  Eigen-level bit parity is unpinned (no Eigen in the image).
"""
import json
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "rng_kat.json")


@pytest.fixture(scope="module")
def kat():
    with open(GOLDEN) as f:
        return json.load(f)


# ------------------------------------------------------------------ RNG (rng.hpp)
def test_derive_seed_matches_reference_binary(orc, kat):
    for s, t, want in kat["derive_seed"]:
        assert orc.derive_seed(int(s), int(t)) == int(want)
    # SURVEY.md §8(c) probe values
    assert orc.derive_seed(1, 1) == 0xF43B3AEEA78D4476
    assert orc.derive_seed(1, 2) == 0x93C5BDBE746B8EA0


@pytest.mark.parametrize("name", ["stream_1", "stream_2", "stream_3"])
def test_streams_match_reference_binary(orc, kat, name):
    st = kat[name]
    seed = int(st["seed"])
    r = orc.Rng(seed)
    assert [r() for _ in st["raw"]] == [int(x) for x in st["raw"]]
    r = orc.Rng(seed)
    assert [r.uniform01() for _ in st["uniform01"]] == st["uniform01"]
    r = orc.Rng(seed)
    assert [r.normal() for _ in st["normal"]] == st["normal"]
    r = orc.Rng(seed)
    assert [r.below(1000003) for _ in st["below_1000003"]] == st["below_1000003"]


# ------------------------------------------------------------ toeplitz.cpp
def test_residual_layout_known_answers(orc):
    # test_toeplitz.cpp:35-51, 154-162
    y = [1, 2, 3, 4, 5]
    assert list(orc.residuals(y, 5, 2, [0, 0])) == [-3, -4, -5]
    assert list(orc.residuals(y, 5, 2, [1, 0])) == [-1, -1, -1]
    a, b = orc.apply_sample(y, 5, 2, [0, 1, 2], [1, 1, 1])
    assert a.tolist() == [[2, 1], [3, 2], [4, 3]] and b.tolist() == [3, 4, 5]
    # single-row edge (test_toeplitz.cpp:53-63)
    a, b = orc.apply_sample([10, 20, 30, 40, 50, 60], 6, 5, [0], [1.0])
    assert a.tolist() == [[50, 40, 30, 20, 10]] and b.tolist() == [60]


def test_residuals_match_dense_definition(orc):
    phi = orc.random_stationary_ar(4, 51)
    y = orc.simulate_ar(phi, 300, 52)
    p = 6
    a, b = orc.apply_sample(y, y.size, p, np.arange(y.size - p), np.ones(y.size - p))
    rphi = np.array([orc.Rng(53).normal() for _ in range(6)])
    assert np.linalg.norm(orc.residuals(y, y.size, p, rphi) - (a @ rphi - b)) < 1e-11
    x, method, _ = orc.solve_exact(a, b)
    r = orc.residuals(y, y.size, p, x)
    assert np.linalg.norm(a.T @ r) <= 1e-8 * np.linalg.norm(a) * (1 + np.linalg.norm(r))


def test_solve_exact_worked_cases(orc):
    x, m, _ = orc.solve_exact(np.eye(2), [3, 4])
    assert np.allclose(x, [3, 4], rtol=1e-14) and m == 0
    x, m, _ = orc.solve_exact(np.ones((3, 1)), [1, 2, 3])
    assert abs(x[0] - 2.0) < 1e-14
    with pytest.raises(orc.OracleError):
        orc.solve_exact(np.zeros((0, 0)), [])


def _randmat(orc, rows, cols, seed):
    r = orc.Rng(seed)
    m = np.empty((rows, cols))
    for i in range(rows):
        for j in range(cols):
            m[i, j] = r.normal()
    return m


def test_solve_exact_vs_normal_equations(orc):
    # test_toeplitz.cpp:118-132
    dims = orc.Rng(31)
    for trial in range(40):
        cols = 1 + dims.below(20)
        rows = cols + 5 + dims.below(175)
        a = _randmat(orc, rows, cols, 1000 + trial)
        b = _randmat(orc, rows, 1, 2000 + trial)[:, 0]
        x, m, _ = orc.solve_exact(a, b)
        ne = np.linalg.solve(a.T @ a, a.T @ b)
        assert np.linalg.norm(x - ne) <= 1e-8 * (1 + np.linalg.norm(ne))
        assert m == 0


def test_rank_deficient_min_norm(orc):
    # test_toeplitz.cpp:134-152: constant series -> rank one, consistent
    y = np.full(9, 2.0)
    a, b = orc.apply_sample(y, 9, 3, np.arange(6), np.ones(6))
    x, m, _ = orc.solve_exact(a, b)
    assert m == 1
    assert np.allclose(x, 1 / 3, rtol=1e-10)
    wide = _randmat(orc, 3, 6, 77)
    bw = _randmat(orc, 3, 1, 78)[:, 0]
    x, m, _ = orc.solve_exact(wide, bw)
    assert m == 1 and np.linalg.norm(wide @ x - bw) < 1e-10
    t = np.linalg.lstsq(wide.T, x, rcond=None)[0]
    assert np.linalg.norm(wide.T @ t - x) < 1e-8


def test_exact_leverage_cases(orc):
    # test_toeplitz.cpp:180-218
    assert np.allclose(orc.exact_leverage([[1.0], [1.0]]), [0.5, 0.5], rtol=1e-14)
    assert np.allclose(orc.exact_leverage([[1.0], [2.0], [3.0]]), np.array([1, 4, 9]) / 14, rtol=1e-13)
    dims = orc.Rng(71)
    for trial in range(10):
        cols = 1 + dims.below(15)
        rows = cols + dims.below(285)
        l = orc.exact_leverage(_randmat(orc, rows, cols, 3000 + trial))
        assert abs(l.sum() - cols) < 1e-8 and l.min() >= -1e-12 and l.max() <= 1 + 1e-12
    dup = _randmat(orc, 10, 1, 81)
    with pytest.raises(orc.OracleError) as e:
        orc.exact_leverage(np.hstack([dup, 2 * dup]))
    assert e.value.code == orc.NUMERICAL


def test_select_order_known_answers(orc):
    # test_toeplitz.cpp:232-251
    bound = 1.96 / math.sqrt(2000.0)
    assert abs(bound - 0.043826932358995874) < 1e-17
    assert orc.select_order([0.9, 0.5, 0.01, 0.005], bound) == 2
    assert orc.select_order([0.01, -0.02, 0.03], 0.05) == 0
    assert orc.select_order([0.9, 0.01, 0.01, 0.01, 0.01, 0.01, 0.05, 0.01], 0.05) == 7
    assert orc.select_order([0.9, -0.06, 0.01], 0.05) == 2


# ------------------------------------------------------------ lsar.cpp
def test_leverage_known_answers(orc):
    # test_lsar.cpp:16-64
    assert np.allclose(orc.init_leverage_p1(np.ones(4)), 0.25, rtol=1e-15)
    assert np.allclose(orc.init_leverage_p1([1, 2, 3]), np.array([1, 4, 9]) / 14, rtol=1e-15)
    with pytest.raises(orc.OracleError) as e:
        orc.init_leverage_p1(np.zeros(3))
    assert e.value.code == orc.NUMERICAL
    nxt = orc.leverage_update([0.1, 0.2], [3, 4])
    assert np.allclose(nxt, [0.46, 0.84], rtol=1e-15)
    with pytest.raises(orc.OracleError) as e:
        orc.leverage_update([0.1, 0.2], [0, 0])
    assert e.value.code == orc.NUMERICAL
    with pytest.raises(orc.OracleError) as e:
        orc.leverage_update([0.1, 0.2], [1, 2, 3])
    assert e.value.code == orc.USAGE
    assert np.allclose(orc.leverage_to_distribution([1, 1, 2]), [0.25, 0.25, 0.5], rtol=1e-15)
    for bad, code in (([0.5, -0.1], orc.USAGE), ([0.0, 0.0], orc.NUMERICAL), ([], orc.USAGE)):
        with pytest.raises(orc.OracleError) as e:
            orc.leverage_to_distribution(bad)
        assert e.value.code == code


def test_recursion_with_exact_residuals_is_exact_leverage(orc):
    # test_lsar.cpp:85-109 and acceptance.cpp:213-245 (criterion 5)
    y = orc.simulate_ar(orc.random_stationary_ar(3, 201), 400, 202)
    p_bar = 8
    w = y.size - p_bar
    s = orc.init_leverage_p1(y[:w])
    for p in range(1, p_bar + 1):
        a, b = orc.apply_sample(y, w + p, p, np.arange(w), np.ones(w))
        exact = orc.exact_leverage(a)
        assert np.max(np.abs(s - exact)) < 1e-10
        assert abs(s.sum() - p) < 1e-10
        if p < p_bar:
            x, _, _ = orc.solve_exact(a, b)
            r = orc.residuals(y, w + p, p, x)
            nxt = orc.leverage_update(s, r)
            assert (nxt - s).min() >= -1e-15
            s = nxt


def test_sample_rows_known_answers(orc):
    # test_sketch.cpp:128-156
    n, c = 16, 8
    idx, w = orc.sample_rows(np.full(n, 1 / n), c, 5)
    assert np.allclose(w, math.sqrt(n / c), rtol=1e-15)
    assert idx.min() >= 0 and idx.max() < n
    point = np.zeros(n); point[3] = 1.0
    idx2, w2 = orc.sample_rows(point, 5, 6)
    assert (idx2 == 3).all() and np.allclose(w2, 1 / math.sqrt(5), rtol=1e-15)
    idx3, _ = orc.sample_rows(np.full(n, 1 / n), c, 5)
    assert (idx3 == idx).all()
    neg = np.full(n, 1 / n); neg[0] = -0.1
    for pi, cc, code in ((neg, c, orc.DATA), (np.full(n, 0.9 / n), c, orc.DATA),
                         (np.full(n, 1 / n), 0, orc.USAGE)):
        with pytest.raises(orc.OracleError) as e:
            orc.sample_rows(pi, cc, 1)
        assert e.value.code == code


def test_apply_sample_known_answers(orc):
    # test_sketch.cpp:176-214
    a, b = orc.apply_sample([1, 2, 3, 4, 5], 5, 2, [1], [0.7])
    assert np.allclose(a, [[0.7 * 3, 0.7 * 2]]) and np.allclose(b, [0.7 * 4])
    a, b = orc.apply_sample([1, 2, 3, 4, 5], 5, 2, [1], [0.7], width=1)
    assert a.shape == (1, 1)
    with pytest.raises(orc.OracleError) as e:
        orc.apply_sample([1, 2, 3, 4, 5], 5, 2, [3], [1.0])
    assert e.value.code == orc.USAGE


def test_compressed_all_rows_equals_exact(orc):
    # test_sketch.cpp:216-250
    y = orc.simulate_ar(orc.random_stationary_ar(3, 31), 200, 32)
    p = 3
    m = y.size - p
    a, b = orc.apply_sample(y, y.size, p, np.arange(m), np.ones(m))
    x, _, _ = orc.solve_exact(a, b)
    a2, b2 = orc.apply_sample(y, y.size, p, np.arange(m), np.full(m, 2.0))
    x2, _, _ = orc.solve_exact(a2, b2)
    assert np.linalg.norm(x2 - x) < 1e-12
    a3, b3 = orc.apply_sample(y, y.size, p, [0, 1], [1.0, 1.0])
    x3, m3, _ = orc.solve_exact(a3, b3)
    assert m3 == 1 and np.isfinite(x3).all()


def test_lsar_fit_recovers_ar2_and_is_deterministic(orc):
    # test_lsar.cpp:171-197
    y = orc.simulate_ar([1.2, -0.36], 6000, 231)
    f = orc.lsar_fit(y, 8, 500, 77)
    assert abs(f.taus[1] + 0.36) < 0.2 and f.p_star >= 2
    assert [c.size for c in f.coefs] == list(range(1, 9))
    g = orc.lsar_fit(y, 8, 500, 77)
    assert (g.taus == f.taus).all()
    h = orc.lsar_fit(y, 8, 500, 78)
    assert not (h.taus == f.taus).all()
    # fixed-index replay reproduces the RNG run exactly
    r = orc.lsar_fit(y, 8, 500, 0, fixed_idx=f.idx, fixed_w=f.w)
    assert (r.taus == f.taus).all()


def test_lsar_fit_errors(orc):
    # test_lsar.cpp:160-169, 199-205
    geo = 0.5 ** np.arange(60)
    with pytest.raises(orc.OracleError) as e:
        orc.lsar_fit(geo, 3, 20, 1)
    assert e.value.code == orc.NUMERICAL
    y = orc.simulate_ar(orc.random_stationary_ar(1, 241), 50, 242)
    for args, code in (((10, 5), orc.USAGE), ((49, 100), orc.DATA), ((0, 100), orc.USAGE)):
        with pytest.raises(orc.OracleError) as e:
            orc.lsar_fit(y, args[0], args[1], 1)
        assert e.value.code == code


# ------------------------------------------------------------ repeated_halving.cpp
def test_generalized_leverage_equals_exact(orc):
    # test_rh.cpp:61-87
    dims = orc.Rng(11)
    for trial in range(6):
        cols = 1 + dims.below(15)
        rows = cols + 1 + dims.below(285)
        a = _randmat(orc, rows, cols, 100 + trial)
        assert np.max(np.abs(orc.generalized_leverage(a, a) - orc.exact_leverage(a))) < 1e-10
    assert np.allclose(orc.generalized_leverage(np.eye(6), np.eye(6)), 1.0, rtol=1e-14)
    c = _randmat(orc, 20, 3, 21)
    with pytest.raises(orc.OracleError) as e:
        orc.generalized_leverage(c, _randmat(orc, 20, 4, 22))
    assert e.value.code == orc.USAGE
    d0 = _randmat(orc, 20, 1, 23)
    dup = np.hstack([d0, d0, _randmat(orc, 20, 1, 24)])
    with pytest.raises(orc.OracleError) as e:
        orc.generalized_leverage(c, dup)
    assert e.value.code == orc.NUMERICAL


def test_sketched_generalized_leverage_concentrates(orc):
    # test_rh.cpp:89-100
    a = _randmat(orc, 512, 8, 31)
    exact = orc.generalized_leverage(a, a)
    approx = orc.generalized_leverage(a, a, 64, 32)
    ratio = approx / exact
    assert ((ratio >= 1 / 3) & (ratio <= 3)).sum() >= 487


def test_rh_defaults(orc):
    # test_rh.cpp:176-194
    cfg = orc.rh_defaults(100000, 9, 500, 13)
    assert cfg.sample_count == 500 and cfg.base_threshold == 500 and cfg.seed == 13
    assert cfg.gaussian_rows == math.ceil(8 * math.log(100000))
    assert orc.lib().orc_default_base_threshold(500, 9) == 500


def test_rh_base_scores_are_exact_leverage(orc):
    # test_rh.cpp:143-155
    y = orc.simulate_ar(orc.random_stationary_ar(2, 61), 60, 62)
    cfg = orc.RhCfg(base_threshold=64, sample_count=32, gaussian_rows=16, seed=5)
    f = orc.rh_fit(y, 4, 32, 1, cfg=cfg)
    a, b = orc.apply_sample(y, y.size, 4, np.arange(56), np.ones(56))
    exact = orc.exact_leverage(np.hstack([a, b[:, None]]))
    assert f.depth == 0
    assert np.max(np.abs(f.scores - exact)) < 1e-10


def test_rh_halving_levels(orc):
    # test_rh.cpp:115-127: 2048 rows, base 256 -> 3 levels; sets sorted, unique
    y = orc.simulate_ar(orc.random_stationary_ar(3, 71), 2052, 72)
    cfg = orc.RhCfg(base_threshold=256, sample_count=256, gaussian_rows=64, seed=9)
    f = orc.rh_fit(y, 4, 256, 3, cfg=cfg, want_levels=True)
    assert f.depth == 3 and list(f.level_sizes) == [2048, 1024, 512, 256]
    prev = np.arange(2048)
    for lvl in f.levels:
        assert (np.diff(lvl) > 0).all() and np.isin(lvl, prev).all()
        prev = lvl
    assert f.scores.min() >= 0 and np.isfinite(f.scores).all()


def test_rh_fit_recovers_ar2(orc):
    # test_rh.cpp:196-221
    y = orc.simulate_ar([1.2, -0.36], 6000, 81)
    f = orc.rh_fit(y, 8, 500, 55)
    assert abs(f.taus[1] + 0.36) < 0.2 and f.p_star >= 2
    g = orc.rh_fit(y, 8, 500, 55)
    assert (g.taus == f.taus).all()
    with pytest.raises(orc.OracleError) as e:
        orc.rh_fit(y, 8, 5, 1)
    assert e.value.code == orc.USAGE

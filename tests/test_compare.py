"""Comparison drivers (bench.cpp:126-243, toeplitz.cpp:140-146): run_compare /
run_sweep over concurrent GPU fits, mirroring test_bench.cpp:121-195."""
import json

import numpy as np
import pytest


def test_trimmed_mean_and_relative_error_cpu():
    import paper_2112_12994_b200 as tf
    assert tf.trimmed_mean([5, 1, 2, 3, 100], 0.2) == (2 + 3 + 5) / 3
    assert tf.trimmed_mean([4.0], 0.0) == 4.0
    with pytest.raises(tf.UsageError):
        tf.trimmed_mean([], 0.0)
    with pytest.raises(tf.UsageError):
        tf.trimmed_mean([1.0], 0.5)
    assert abs(tf.relative_error_pct([1, 2], [1, 1]) - 100 * np.sqrt(0.5)) < 1e-12
    with pytest.raises(tf.UsageError):
        tf.relative_error_pct([1, 2, 3], [1, 1])
    with pytest.raises(tf.NumericalError):
        tf.relative_error_pct([1, 2], [0, 0])


def test_report_writers_cpu(tmp_path):
    import paper_2112_12994_b200 as tf
    pacf = tf.PACFResult(taus=[0.4, -0.2, 0.05], bound=0.1, method="lsar")
    p = tmp_path / "plot.csv"
    tf.write_pacf_plot_csv(pacf, str(p))
    assert p.read_text().splitlines() == ["lag,tau,bound_hi,bound_lo", "1,0.40000000000000002,0.10000000000000001,-0.10000000000000001",
                                          "2,-0.20000000000000001,0.10000000000000001,-0.10000000000000001",
                                          "3,0.050000000000000003,0.10000000000000001,-0.10000000000000001"]
    tf.write_pacf_csv(pacf, str(tmp_path / "pacf.csv"))
    assert (tmp_path / "pacf.csv").read_text().splitlines()[0] == "lag,tau,bound"
    rows = [tf.SweepRow("lsar", 200, 0.0, 1.5), tf.SweepRow("rh", 200, 0.0, 2.5)]
    tf.write_sweep_csv(rows, str(tmp_path / "sweep.csv"))
    assert (tmp_path / "sweep.csv").read_text().splitlines() == ["method,c,max_seconds,max_error_pct",
                                                                 "lsar,200,0,1.5", "rh,200,0,2.5"]
    with pytest.raises(tf.DataError, match="cannot write"):
        tf.write_pacf_csv(pacf, str(tmp_path / "no" / "such" / "dir.csv"))


def _series():
    from paper_2112_12994_b200 import gen
    return gen.simulate_roots(gen.ar_roots(4, 1.3, 3.0, 8), 3000, 8)


@pytest.mark.gpu
def test_run_compare_aggregates_repetitions():
    import paper_2112_12994_b200 as tf
    s = tf.TimeSeries(_series())
    rep = tf.run_compare(s, 5, 300, 3, 0.0, 21, False, workers=3)
    assert rep.n == 3000 and rep.repetitions == 3 and len(rep.exact_taus) == 5
    assert len(rep.lsar.trimmed_error_pct) == 5 and len(rep.rh.trimmed_error_pct) == 5
    assert len(rep.lsar.p_stars) == 3 and len(rep.rh.p_stars) == 3
    assert all(np.isfinite(e) and e >= 0 for e in rep.lsar.trimmed_error_pct + rep.rh.trimmed_error_pct)
    assert rep.lsar.mean_lag_seconds == [0.0] * 5  # timing disabled
    # one repetition, no trimming: that run's direct error (test_bench.cpp:136-144)
    single = tf.run_compare(s, 5, 300, 1, 0.0, 21, False)
    exact = tf.exact_fit(s, 5)
    one = tf.lsar_fit_batch(s, 5, 300, [tf.derive_seed(21, 0x1000)])[0]  # the repetitions' batched path
    for h in range(5):
        direct = tf.relative_error_pct(one.per_lag_coefficients[h], exact.per_lag_coefficients[h])
        assert abs(single.lsar.trimmed_error_pct[h] - direct) <= 1e-12 * max(direct, 1e-300)
    # the concurrent repetitions equal sequential fits with the same seeds
    for r in range(3):
        f = tf.rh_fit(s, 5, 300, None, tf.derive_seed(21, 0x2000 + r))
        assert rep.rh.p_stars[r] == f.p_star
    j = json.loads(tf.compare_to_json(rep))
    assert j["n"] == 3000 and j["exact"]["p_star"] == rep.exact_p_star
    assert len(j["lsar"]["trimmed_error_pct"]) == 5 and len(j["rh"]["p_stars"]) == 3
    assert tf.compare_to_json(rep) == tf.compare_to_json(rep)
    import os, tempfile
    d = tempfile.mkdtemp()
    tf.write_compare_errors_csv(rep, os.path.join(d, "e.csv"))
    tf.write_compare_timing_csv(rep, os.path.join(d, "t.csv"))
    assert open(os.path.join(d, "e.csv")).readline().strip() == "lag,lsar_error,rh_error"
    assert open(os.path.join(d, "t.csv")).readline().strip() == "lag,exact_cum,lsar_cum,rh_cum"
    with pytest.raises(tf.UsageError):
        tf.run_compare(s, 5, 300, 0, 0.0, 1)
    with pytest.raises(tf.UsageError):
        tf.run_compare(s, 5, 300, 1, 0.7, 1)


@pytest.mark.gpu
def test_run_sweep_rows():
    import paper_2112_12994_b200 as tf
    s = tf.TimeSeries(_series())
    rows = tf.run_sweep(s, [200, 400], 4, 2, 0.0, 41, False, workers=2)
    assert [(r.method, r.c) for r in rows] == [("lsar", 200), ("rh", 200), ("lsar", 400), ("rh", 400)]
    assert all(np.isfinite(r.max_error_pct) and r.max_error_pct >= 0 and r.max_lag_seconds == 0.0 for r in rows)
    with pytest.raises(tf.UsageError):
        tf.run_sweep(s, [], 4, 2, 0.0, 1)

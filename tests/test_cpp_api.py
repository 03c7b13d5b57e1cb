"""The C++ host API (include/toepfit_b200.hpp) gives the same fits as the
Python mirror (both call the same C ABI) and maps statuses to the reference's
exception types."""
import json
import subprocess

import numpy as np
import pytest


def test_cpp_header_compiles():
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.check_call(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(root, "include"),
                           os.path.join(root, "tests", "cpp", "test_cpp_api.cpp")])


@pytest.mark.gpu
def test_cpp_api_matches_python(tmp_path):
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import build, gen
    exe = build.build_cpp_api_test()
    roots = gen.ar_roots(8, 1.2, 3.0, 4)
    y = gen.simulate_roots(roots, 30000, 4)
    f = tmp_path / "y.bin"
    y.astype("<f8").tofile(f)
    out = subprocess.run([exe, str(f), "16", "900", "11"], capture_output=True, text=True, check=True)
    res = json.loads(out.stdout)
    eng = tf.Engine(0)
    s = tf.TimeSeries(y)
    a = tf.lsar_fit(s, 16, 900, 11, engine=eng)
    b = tf.rh_fit(s, 16, 900, None, 11, engine=eng)
    assert res["lsar"]["taus"] == a.pacf.taus and res["lsar"]["p_star"] == a.p_star
    assert res["rh"]["taus"] == b.pacf.taus and res["rh"]["p_star"] == b.p_star
    assert res["lsar"]["select"] == a.p_star
    sr = tf.srht_fit(s, 16, 900, 11, engine=eng)
    ex = tf.exact_fit(s, 16, engine=eng)
    assert res["srht"]["taus"] == sr.pacf.taus and res["srht"]["p_star"] == sr.p_star
    assert res["exact"]["taus"] == ex.pacf.taus and res["exact"]["p_star"] == ex.p_star
    assert res["errors"] == {"usage": 1, "data": 1, "numerical": 1}
    bt = tf.lsar_fit_batch(s, 16, 900, [11, 12], engine=eng)
    assert res["batch0"]["taus"] == bt[0].pacf.taus and res["batch1"]["taus"] == bt[1].pacf.taus
    assert res["batch0"]["p_star"] == bt[0].p_star
    rs = res["rowsource"]
    assert rs["levels"] == 2 and rs["rows"] == 128 and abs(rs["lev_sum"] - 6.0) < 1e-10  # exact leverage sums to k
    drv = res["driver"]
    assert drv["rows"] == y.size - 16 and drv["m1"] == y.size - 15 and drv["m2"] == y.size - 14 and drv["p2"] == 2
    assert abs(drv["ssum2"] - 2.0) < 1e-12 and drv["replay"] == 1
    d = tf.LsarDriver(s, 16, 900, 11, engine=eng)
    st2 = d.advance(d.first_lag())
    assert np.allclose(drv["phi2"], st2.coefficients, rtol=1e-9, atol=0)
    eng.close()

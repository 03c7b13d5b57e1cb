"""CPU-side checks of the drop-in boundary: the in-tree C-ABI library loads,
exports exactly what include/toepfit_b200.h declares, and its host-only
entry points behave like the reference (no GPU calls here)."""
import ctypes as C
import json
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "toepfit_b200.h")


@pytest.fixture(scope="module")
def abi():
    import __graft_entry__ as g
    from paper_2112_12994_b200 import build as b
    b.build()
    from paper_2112_12994_b200 import _abi
    return _abi


def declared_functions():
    text = open(HEADER).read()
    pat = r"^\s*(?:const\s+char\s*\*|tf_status|void|int|int64_t|uint64_t)\s+(tf_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(pat, text, flags=re.M)))


def test_library_exports_every_declared_symbol(abi):
    L = abi.lib()
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(abi.EXPORTS)


def test_sm100a_code_in_library(abi):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_derive_seed_matches_reference_golden(abi):
    L = abi.lib()
    kat = json.load(open(os.path.join(ROOT, "tests", "golden", "rng_kat.json")))
    for s, t, want in kat["derive_seed"]:
        assert L.tf_derive_seed(int(s), int(t)) == int(want)


def test_select_order_known_answers(abi):
    # test_toeplitz.cpp:232-251
    L = abi.lib()

    def so(t, b):
        a = np.ascontiguousarray(t, dtype=np.float64)
        return L.tf_select_order(abi.ptr(a), a.size, b)

    assert so([0.9, 0.5, 0.01, 0.005], 1.96 / math.sqrt(2000.0)) == 2
    assert so([0.01, -0.02, 0.03], 0.05) == 0
    assert so([0.9, 0.01, 0.01, 0.01, 0.01, 0.01, 0.05, 0.01], 0.05) == 7
    assert so([0.9, -0.06, 0.01], 0.05) == 2


def test_create_without_gpu_fails_loudly(abi):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = C.c_void_p()
    opts = abi.TfOpts(device=0, priority=0)
    assert abi.lib().tf_create(C.byref(opts), C.byref(ctx)) == abi.TF_CUDA
    import paper_2112_12994_b200 as tf
    with pytest.raises(tf.CudaError):
        tf.Engine(0)


def test_host_mirror_validation():
    import paper_2112_12994_b200 as tf
    with pytest.raises(tf.DataError):
        tf.TimeSeries([])
    with pytest.raises(tf.DataError):
        tf.TimeSeries([1.0, float("nan")])
    cfg = tf.RHConfig.defaults(100000, 9, 500, 13)  # test_rh.cpp:176-194
    assert cfg.base_threshold == 500 and cfg.gaussian_rows == math.ceil(8 * math.log(100000))
    bad = tf.RHConfig(base_threshold=10, sample_count=20, gaussian_rows=3)
    with pytest.raises(tf.UsageError):
        bad.validate()
    with pytest.raises(tf.UsageError):  # argument errors come before any device work
        tf.run_fit(tf.TimeSeries([1.0, 2.0, 3.0]), "srht", 1, 0, 0)
    with pytest.raises(tf.UsageError):
        tf.run_fit(tf.TimeSeries([1.0, 2.0, 3.0]), "nope", 1, 10, 0)
    # sample count formula: the reference's frozen regression value (test_sketch.cpp:112-125)
    sc = tf.srht_sample_count(1 << 20, 10, 0.5)
    assert abs(sc.formula_value - 6633578.924774391) <= 1e-12 * 6633578.924774391
    assert sc.capped and sc.c == 1 << 20
    assert tf.srht_sample_count(1 << 20, 10, 0.9).formula_value <= sc.formula_value
    for args in ((5, 5, 0.5), (10, 0, 0.5), (100, 5, 0.0), (100, 5, 1.0)):
        with pytest.raises(tf.UsageError):
            tf.srht_sample_count(*args)
    with pytest.raises(tf.UsageError):
        tf.run_fit(tf.TimeSeries([1.0, 2.0, 3.0]), "lsar", 1, 0, 0)


def test_report_json_schema():
    import paper_2112_12994_b200 as tf
    r = tf.RunReport(method="lsar", n=10, p_bar=2, c=5, seed=1, timing_recorded=False,
                     upfront_seconds=0.0, per_lag_seconds=[0.0, 0.0], cumulative_seconds=[0.0, 0.0],
                     pacf=tf.PACFResult([0.5, -0.1], 0.2, "lsar"), p_star=1, coefficients=[0.5])
    j = json.loads(tf.report_to_json(r))
    assert list(j) == sorted(["method", "n", "p_bar", "c", "seed", "timing_recorded",
                              "upfront_seconds", "per_lag_seconds", "cumulative_seconds", "pacf",
                              "p_star", "coefficients"])
    assert j["pacf"] == {"bound": 0.2, "method": "lsar", "taus": [0.5, -0.1]}


def test_generator_reproducible_and_shaped():
    from paper_2112_12994_b200 import gen
    assert gen._derive_py(1, 1) == 0xF43B3AEEA78D4476
    y1, phi, p_bar, cs = gen.make_config_series("C1", n=5000)
    y2, _, _, _ = gen.make_config_series("C1", n=5000)
    assert (y1 == y2).all() and y1.size == 5000 and phi.size == 20 and p_bar == 100
    y3, _, _, _ = gen.make_config_series("C3", n=20000)
    assert np.isfinite(y3).all()

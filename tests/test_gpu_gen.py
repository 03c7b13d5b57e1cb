"""On-device synthetic series (tf_generate_series):
pinned against a host restatement of the same generator (counter-RNG
Box-Muller innovations, sequential first-order sections)."""
import math

import numpy as np
import pytest
from scipy.signal import lfilter

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def host_innovations(seed, total):
    t = np.arange(total + (total & 1), dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) + (t + np.uint64(1)) * np.uint64(GOLD)).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u1 = u[0::2] + 2.0 ** -54
    u2 = u[1::2]
    rad = np.sqrt(-2.0 * np.log(u1))
    out = np.empty(u.size)
    out[0::2] = rad * np.cos(2 * np.pi * u2)
    out[1::2] = rad * np.sin(2 * np.pi * u2)
    return out[:total]


def test_generated_series_matches_host_restatement():
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen
    eng = tf.Engine(0)
    roots = gen.ar_roots(6, 1.2, 3.0, 17)
    n, burn, seed = 60000, 1000, 12345
    eng.generate_series(roots, n, seed, burn_in=burn)
    y = eng.download_series(n)
    x = host_innovations(seed, n + burn)
    for r in roots:
        x = lfilter([1.0], [1.0, -1.0 / r], x)
    ref = x[burn:]
    assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-9
    eng.close()


def test_generated_series_fits_its_ar_model():
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen
    eng = tf.Engine(0)
    roots = gen.ar_roots(4, 1.3, 2.5, 5)
    eng.generate_series(roots, 400000, 7)
    taus, coefs, _, _ = eng.exact_sweep(4)
    phi = np.array(tf.api._unpack(coefs, 4)[3])
    assert np.max(np.abs(phi - gen.ar_coefficients(roots))) < 0.02
    # heavy-tailed innovations have unit variance and fat tails
    eng.generate_series([], 400000, 9, innovations="t3", burn_in=0)
    e = eng.download_series(400000)
    assert abs(np.var(e) - 1.0) < 0.1
    assert np.mean(e ** 4) / np.var(e) ** 2 > 5.0
    eng.close()

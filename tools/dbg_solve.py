"""Standalone sampled solves at several lags (method codes / failures)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
eng = tf.Engine(0)
for p in [33, 100, 200, 216, 230, 300]:
    y = gen.simulate_roots(gen.ar_roots(20, 1.2, 3.0, p), 60000, p)
    rng = np.random.default_rng(p)
    c = max(4 * p, 600)
    idx = rng.integers(0, y.size - p, size=c)
    w = rng.uniform(0.5, 2.0, size=c)
    try:
        phi, method = eng.solve_sampled(y, y.size, p, idx, w)
        print(p, "method", method, "phi[0]", phi[0])
    except Exception as e:
        print(p, "ERR", e)

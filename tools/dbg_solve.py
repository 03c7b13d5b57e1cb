import sys, numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
from oracle import oracle as orc
eng = tf.Engine(0)
for p in [5, 31, 32, 33, 63, 64, 100, 200, 300]:
    roots = gen.ar_roots(20, 1.2, 3.0, p); y = gen.simulate_roots(roots, 60000, p)
    rng = np.random.default_rng(p); c = max(4 * p, 600)
    idx = rng.integers(0, y.size - p, size=c); w = rng.uniform(0.5, 2.0, size=c)
    try:
        phi, m = eng.solve_sampled(y, y.size, p, idx, w)
    except Exception as e:
        print(p, "ERR", e); continue
    a, b = orc.apply_sample(y, y.size, p, idx, w); ref, _, _ = orc.solve_exact(a, b)
    print(p, "method", m, "relerr %.2e" % (np.max(np.abs(phi - ref)) / np.max(np.abs(ref))), "cond %.2e" % np.linalg.cond(a))
y, _, p_bar, _ = gen.make_config_series("C2", n=2_000_000)
try:
    fit = tf.lsar_fit(tf.TimeSeries(y), 60, 10000, 1, engine=eng, want_diag=True)
    print("sweep ok; methods", np.bincount(fit.diag["method"]))
except Exception as e:
    print("sweep ERR", e)

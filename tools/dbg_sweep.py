import sys, numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
eng = tf.Engine(0)
y, _, p_bar, _ = gen.make_config_series("C2")
for c in [10000, 100000]:
    try:
        fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, c, 1, engine=eng, want_diag=True)
        print(c, "sweep ok; methods", np.bincount(fit.diag["method"]), "ms", sum(fit.per_lag_seconds)*1e3)
    except Exception as e:
        print(c, "sweep ERR", e)

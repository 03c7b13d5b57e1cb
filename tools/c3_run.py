"""BASELINE C3: heavy-tailed AR(50) (t3 innovations, 1 % +-10 sigma outliers), n = 1e8,
LSAR p = 1..200 with s = 1e5 on one GPU (device time per phase)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
t0 = time.time()
y, _, p_bar, cs = gen.make_config_series("C3")
print(f"generated n={y.size} in {time.time() - t0:.1f} s", flush=True)
eng = tf.Engine(0)
s = tf.TimeSeries(y)
for rep in range(2):
    fit = tf.lsar_fit(s, p_bar, cs[0], 1 + rep, engine=eng, want_diag=True)
    ph = fit.diag["phases"].sum(0)
    tot = sum(fit.per_lag_seconds)
    print(f"C3 LSAR sweep {tot:.3f} s device (sample {ph[0]:.3f}, solve {ph[1]:.3f}, pass {ph[2]:.3f}); "
          f"{p_bar * (y.size - p_bar) / tot:.3e} rows*orders/s; p*={fit.p_star}; methods {np.bincount(fit.diag['method'])}")

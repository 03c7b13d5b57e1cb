"""C4 shape check (p_bar = 500, s = 2e5, AR(100) roots in [1.05, 2]) on a shorter series."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
y, _, p_bar, cs = gen.make_config_series("C4", n=n)
eng = tf.Engine(0)
t0 = time.time()
fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, cs[0], 1, engine=eng, want_diag=True)
dt = time.time() - t0
ph = fit.diag["phases"]
print(f"C4-shape n={n} p_bar={p_bar} c={cs[0]}: device {sum(fit.per_lag_seconds):.3f} s (wall {dt:.2f}), p*={fit.p_star}, "
      f"methods {np.bincount(fit.diag['method'])}, phases sample/solve/pass {ph.sum(0)}")
for p in [100, 250, 400, 500]:
    print(f"  p={p}: solve {ph[p-1,1]*1e3:.2f} ms pass {ph[p-1,2]*1e3:.2f} ms")

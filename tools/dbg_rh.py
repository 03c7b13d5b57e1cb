import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
eng = tf.Engine(0)
y, _, p_bar, _ = gen.make_config_series("C2")
ts = tf.TimeSeries(y)
for c in [10000, 100000]:
    for rep in range(2):
        t0 = time.time()
        fit = tf.rh_fit(ts, p_bar, c, None, 1 + rep, engine=eng, want_diag=(rep == 0))
        wall = time.time() - t0
        print(f"rh c={c} upfront {fit.upfront_seconds*1e3:.2f} ms lags {sum(fit.per_lag_seconds)*1e3:.2f} ms "
              f"wall {wall*1e3:.0f} ms p*={fit.p_star} depth={fit.diag['depth'] if fit.diag else '-'}")
    f2 = tf.lsar_fit(ts, p_bar, c, 1, engine=eng)
    print(f"lsar c={c} {sum(f2.per_lag_seconds)*1e3:.2f} ms p*={f2.p_star}")

import sys
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
eng = tf.Engine(0)
y, _, p_bar, _ = gen.make_config_series("C2")
c = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
fit = tf.rh_fit(tf.TimeSeries(y), p_bar, c, None, 1, engine=eng)
print("upfront ms", fit.upfront_seconds * 1e3, "lags ms", sum(fit.per_lag_seconds) * 1e3)

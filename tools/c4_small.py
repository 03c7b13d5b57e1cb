import sys
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
y, _, p_bar, cs = gen.make_config_series("C4", n=2_000_000)
fit = tf.lsar_fit(tf.TimeSeries(y), p_bar, cs[0], 1, engine=tf.Engine(0))
print(sum(fit.per_lag_seconds))

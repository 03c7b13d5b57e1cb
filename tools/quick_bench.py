"""Quick timing of one LSAR sweep (development helper)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
t0 = time.time()
y, phi_true, p_bar, cs = gen.make_config_series(name, n=n)
print(f"gen {name} n={y.size} in {time.time()-t0:.1f}s", flush=True)
eng = tf.Engine(0)
s = tf.TimeSeries(y)
for rep in range(3):
    t0 = time.time()
    fit = tf.lsar_fit(s, p_bar, c, 1 + rep, engine=eng, want_diag=(rep == 2))
    wall = time.time() - t0
    dev = sum(fit.per_lag_seconds)
    ro = p_bar * (y.size - p_bar)
    print(f"rep {rep}: wall {wall*1e3:.1f} ms  device {dev*1e3:.1f} ms  rows*orders/s {ro/dev:.3e}  p* {fit.p_star}", flush=True)
lag = np.array(fit.per_lag_seconds) * 1e6
print("per-lag us: p=1 %.0f p=10 %.0f p=50 %.0f p=100 %.0f p=last %.0f" % (lag[0], lag[min(9,p_bar-1)], lag[min(49,p_bar-1)], lag[min(99,p_bar-1)], lag[-1]))
print("methods:", np.bincount(fit.diag["method"]))
print("taus[:5]", np.array(fit.pacf.taus[:5]), "true phi[:5]", phi_true[:5])

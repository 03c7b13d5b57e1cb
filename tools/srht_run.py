"""SRHT sweep at BASELINE scales on one GPU, plus the
oracle's per-lag time on a few lags for comparison (development helper).
usage: python tools/srht_run.py [C1|C2] [--oracle-lags 1,50,100]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
y, _, p_bar, cs = gen.make_config_series(name)
c = cs[0]
eng = tf.Engine(0)
s = tf.TimeSeries(y)
for rep in range(2):
    t0 = time.time()
    fit = tf.srht_fit(s, p_bar, c, 1 + rep, engine=eng)
    dev = sum(fit.per_lag_seconds)
    print(f"{name} SRHT n={y.size} p_bar={p_bar} c={c}: device {dev:.3f} s (wall {time.time() - t0:.2f} s), "
          f"{p_bar * (y.size - p_bar) / dev:.3e} rows*orders/s, p*={fit.p_star}, "
          f"lag 1 {fit.per_lag_seconds[0] * 1e3:.2f} ms, lag {p_bar} {fit.per_lag_seconds[-1] * 1e3:.2f} ms", flush=True)
if "--oracle-lags" in sys.argv:
    import ctypes as C
    from oracle import oracle as orc
    lags = [int(v) for v in sys.argv[sys.argv.index("--oracle-lags") + 1].split(",")]
    for h in lags:
        m = y.size - h
        a = np.empty((m, h), order="F")
        for j in range(h):
            a[:, j] = y[h - 1 - j:h - 1 - j + m]
        t0 = time.time()
        orc.srht_solve(a, y[h:h + m], c, tf.derive_seed(1, h))
        print(f"oracle srht_solve lag {h}: {time.time() - t0:.2f} s (1 thread)", flush=True)

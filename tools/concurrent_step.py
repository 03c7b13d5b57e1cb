"""The four C2 sweeps sequentially vs concurrently (one context + stream each)."""
import sys, time, threading
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
y, _, p_bar, cs = gen.make_config_series("C2")
sweeps = [("lsar", c) for c in cs] + [("rh", c) for c in cs]
engs = [tf.Engine(0) for _ in sweeps]
ts = tf.TimeSeries(y)
def run(i, seed):
    m, c = sweeps[i]
    if m == "lsar":
        f = tf.lsar_fit(ts, p_bar, c, seed + i, engine=engs[i])
    else:
        f = tf.rh_fit(ts, p_bar, c, None, seed + i, engine=engs[i])
    return f
for rep in range(3):
    # sequential
    t0 = time.time()
    dev = 0.0
    for i in range(4):
        f = run(i, 10 * rep)
        dev += sum(f.per_lag_seconds) + f.upfront_seconds
    seq_wall = time.time() - t0
    # concurrent
    t0 = time.time()
    th = [threading.Thread(target=run, args=(i, 10 * rep)) for i in range(4)]
    for t in th: t.start()
    for t in th: t.join()
    conc_wall = time.time() - t0
    spans = [e.sweep_span(engs[0]) for e in engs]
    region = max(b for a, b in spans) - min(a for a, b in spans)
    print(f"rep {rep}: sequential device {dev*1e3:.1f} ms (wall {seq_wall*1e3:.0f}); concurrent region {region:.1f} ms (wall {conc_wall*1e3:.0f}) spans {[(round(a,1), round(b,1)) for a,b in spans]}")

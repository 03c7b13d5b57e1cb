"""The four C2 sweeps concurrently (one context + stream each) with stream
priorities per sweep: which assignment shortens the step (the sweeps share
the GPU; the longest chain should not wait behind the others' big kernels)."""
import sys, threading
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
y, _, p_bar, cs = gen.make_config_series("C2")
sweeps = [("lsar", c) for c in cs] + [("rh", c) for c in cs]
ts = tf.TimeSeries(y)
assignments = {"none": [0, 0, 0, 0], "rh1e5": [0, 0, 0, 2], "rh>lsar": [0, 1, 2, 3],
               "lsar>rh": [3, 2, 1, 0], "rh": [0, 0, 2, 2], "small first": [3, 1, 2, 0]}
for name, prios in assignments.items():
    engs = [tf.Engine(0, priority=p) for p in prios]
    def run(i, seed):
        m, c = sweeps[i]
        if m == "lsar":
            tf.lsar_fit(ts, p_bar, c, seed + i, engine=engs[i])
        else:
            tf.rh_fit(ts, p_bar, c, None, seed + i, engine=engs[i])
    res = []
    for rep in range(4):
        th = [threading.Thread(target=run, args=(i, 10 * rep)) for i in range(4)]
        for t in th: t.start()
        for t in th: t.join()
        spans = [e.sweep_span(engs[0]) for e in engs]
        region = max(b for a, b in spans) - min(a for a, b in spans)
        if rep >= 2:
            res.append((round(region, 1), [round(b, 1) for a, b in spans]))
    print(f"{name:12s} prios {prios}: {res}", flush=True)
    for e in engs:
        e.close()

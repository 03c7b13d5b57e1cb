"""One C2 bench step (4 sweeps) on a warmed engine, wrapped in cudaProfilerStart/Stop."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
eng = tf.Engine(0)
y, _, p_bar, cs = gen.make_config_series("C2")
ts = tf.TimeSeries(y)
sweeps = [("lsar", c) for c in cs] + [("rh", c) for c in cs]
def step(seed):
    tot = 0.0
    for k, (m, c) in enumerate(sweeps):
        f = (tf.lsar_fit(ts, p_bar, c, seed + k, engine=eng) if m == "lsar"
             else tf.rh_fit(ts, p_bar, c, None, seed + k, engine=eng))
        t = sum(f.per_lag_seconds) + f.upfront_seconds
        print(m, c, f"{t*1e3:.1f} ms", flush=True)
        tot += t
    return tot
step(1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
print("step ms", step(2) * 1e3)
torch.cuda.synchronize()
torch.cuda.profiler.stop()

"""One batched C5-shape sweep (256 series) inside cudaProfilerStart/Stop, for ncu launch lists."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
nser = int(sys.argv[1]) if len(sys.argv) > 1 else 256
Y = np.stack([gen.simulate_roots(gen.ar_roots(1 + k % 10, 1.1, 3.0, 1000 + k), 100_000, 1000 + k) for k in range(nser)])
eng = tf.Engine(0)
tf.lsar_fit_batch(Y, 50, 2000, list(range(nser)), engine=eng)
torch.cuda.synchronize()
torch.cuda.profiler.start()
f = tf.lsar_fit_batch(Y, 50, 2000, list(range(nser)), engine=eng)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("device lag loop s", sum(f[0].per_lag_seconds))

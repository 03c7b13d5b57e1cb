"""One sampled solve at lag p (for ncu captures of the solve kernels)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen

p = int(sys.argv[1]) if len(sys.argv) > 1 else 200
c = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
y, _, _, _ = gen.make_config_series("C2", n=2_000_000)
rng = np.random.default_rng(1)
idx = rng.integers(0, y.size - p, size=c)
w = np.ones(c)
eng = tf.Engine(0)
for _ in range(2):
    phi, m = eng.solve_sampled(y, y.size, p, idx, w)
print("method", m, "phi[:3]", phi[:3])

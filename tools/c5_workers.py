import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
nser = int(sys.argv[1])
rng = np.random.default_rng(2112)
ys = []
for k in range(nser):
    q = int(rng.integers(1, 11))
    ys.append(gen.simulate_roots(gen.ar_roots(q, 1.1, 3.0, 1000 + k), 100_000, 1000 + k))
for workers in [int(x) for x in sys.argv[2].split(",")]:
    tf.fit_many(ys[:workers*2], "lsar", 50, 2000, list(range(workers*2)), workers=workers)  # warm (graphs per context)
    t0 = time.time()
    fits = tf.fit_many(ys, "lsar", 50, 2000, list(range(nser)), workers=workers)
    dt = time.time() - t0
    print(f"workers {workers}: {dt:.2f} s, {dt / nser * 1e3:.3f} ms/series", flush=True)

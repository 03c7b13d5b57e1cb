"""BASELINE C5: 4096 independent series (n = 1e5, AR order 1..10, roots in
[1.1, 3]), batched LSAR p = 1..50 with s = 2000 -- fit_many over concurrent
contexts on one GPU (a subset by default; --all for the full batch)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
nser = 4096 if "--all" in sys.argv else 256
rng = np.random.default_rng(2112)
ys = []
for k in range(nser):
    q = int(rng.integers(1, 11))
    ys.append(gen.simulate_roots(gen.ar_roots(q, 1.1, 3.0, 1000 + k), 100_000, 1000 + k))
for workers in (8, 16):
    tf.fit_many(ys[:16], "lsar", 50, 2000, list(range(16)), workers=workers)  # warm
    t0 = time.time()
    fits = tf.fit_many(ys, "lsar", 50, 2000, list(range(nser)), workers=workers)
    dt = time.time() - t0
    ro = nser * 50 * (100_000 - 50)
    print(f"C5 {nser} series, workers {workers}: {dt:.2f} s wall, {ro / dt:.3e} rows*orders/s, "
          f"{dt / nser * 1e3:.2f} ms/series")

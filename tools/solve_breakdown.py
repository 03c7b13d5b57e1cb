"""Per-kernel cost of one C4-shaped sampled solve (c = 2e5 rows of a C4
series, log-normal weights) at several lag orders: run plain for wall times,
under `ncu --metrics gpu__time_duration.sum --csv` for the kernel split
(tools/ncu_summary.py groups it)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf  # noqa: E402
from paper_2112_12994_b200 import gen  # noqa: E402

ps = [int(a) for a in sys.argv[1:]] or [50, 150, 300, 500]
c = 200_000
y, _, _, _ = gen.make_config_series("C4", n=4_000_000)
rng = np.random.default_rng(1)
eng = tf.Engine(0)
for p in ps:
    idx = rng.integers(0, y.size - p, size=c)
    w = np.exp(rng.normal(size=c))
    eng.solve_sampled(y, y.size, p, idx, w)
    t0 = time.perf_counter()
    phi, m = eng.solve_sampled(y, y.size, p, idx, w)
    print(f"p {p}: method {m} wall {1e3 * (time.perf_counter() - t0):.2f} ms (incl. upload of y and the draws)")

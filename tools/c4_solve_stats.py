"""Per-lag rank and min-norm SVD sweep counts of a C4-shaped sweep (the solve
does not depend on n: c = 2e5, p_bar = 500).  python tools/c4_solve_stats.py [n]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf  # noqa: E402
from paper_2112_12994_b200 import gen  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000_000
eng = tf.Engine(0)
eng.generate_series(gen.ar_roots(100, 1.05, 2.0, 2112_12994), n, 2112_12994, "normal")
out = eng.lsar_sweep(500, 200_000, 1, want_diag="light", n=n)
d = out[4]
for lo in range(0, 500, 50):
    sl = slice(lo, lo + 50)
    print(f"lags {lo + 1:3d}-{lo + 50:3d}: rank {d['rank'][sl].min():4d}-{d['rank'][sl].max():4d}  "
          f"svd sweeps {d['svd_sweeps'][sl].min():2d}-{d['svd_sweeps'][sl].max():2d} "
          f"(mean {d['svd_sweeps'][sl].mean():.1f})  solve ms {1e3 * d['phases'][sl, 1].mean():.2f}")

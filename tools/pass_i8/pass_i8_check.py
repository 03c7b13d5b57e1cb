"""INT8 tensor-core pass vs the fp64 DMMA pass on one series: the same
fixed draws (the DMMA run's indices and weights) through both, then the
per-lag window residual norms, taus and p* side by side, and the sweep time
of each.  usage: python tools/pass_i8_check.py [C1|C2|C4] [n] [p_bar] [c]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf  # noqa: E402
from paper_2112_12994_b200 import gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else None
y, _, pb, cs = gen.make_config_series(cfg, n=n)
pb = int(sys.argv[3]) if len(sys.argv) > 3 else pb
c = int(sys.argv[4]) if len(sys.argv) > 4 else cs[0]
print(f"{cfg}: n {y.size} p_bar {pb} c {c} max|y|/rms {np.max(np.abs(y)) / np.sqrt(np.mean(y * y)):.1f}")
res = {}
for mode in ["dmma", "i8"]:
    os.environ["TF_PASS"] = mode
    eng = tf.Engine(0)
    kw = {}
    if mode == "i8":
        kw = dict(fixed_idx=res["dmma"].diag["idx"], fixed_w=res["dmma"].diag["w"])
    fit = tf.lsar_fit(tf.TimeSeries(y), pb, c, 7, engine=eng, want_diag=True, **kw)
    t0 = time.perf_counter()
    fit2 = tf.lsar_fit(tf.TimeSeries(y), pb, c, 7, engine=eng, want_diag=True, **kw)
    dt = time.perf_counter() - t0
    res[mode] = fit
    print(f"{mode}: p* {fit.p_star} wall {dt:.3f} s  device sweep {sum(fit2.per_lag_seconds):.3f} s")
    eng.close()
a, b = res["dmma"], res["i8"]
ra, rb = a.diag["rnorm2"], b.diag["rnorm2"]
print("window ||r||^2 rel diff: max", float(np.max(np.abs(rb / ra - 1))), "per decile",
      [f"{float(np.max(np.abs(rb[k:k + pb // 10] / ra[k:k + pb // 10] - 1))):.1e}" for k in range(0, pb, max(1, pb // 10))])
ta, tb = np.asarray(a.pacf.taus), np.asarray(b.pacf.taus)
print("tau max abs diff", float(np.max(np.abs(ta - tb))), " ssum rel diff", float(np.max(np.abs(b.diag["ssum"] / a.diag["ssum"] - 1))))
print("p*", a.p_star, b.p_star)

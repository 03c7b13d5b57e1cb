"""BASELINE C4 at full size on one GPU: AR(100), roots |r| in [1.05, 2], n = 1e9
(8 GB), generated on the device (tf_generate_series), LSAR p = 1..500, s = 2e5."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
q, lo, hi, _, p_bar, cs, _, _ = gen.CONFIGS["C4"]
roots = gen.ar_roots(q, lo, hi, 2112_12994)
eng = tf.Engine(0)
t0 = time.time()
eng.generate_series(roots, n, 2112_12994)
print(f"generated n={n} on the device in {time.time() - t0:.2f} s", flush=True)
t0 = time.time()
taus, coefs, secs, pstar, diag = eng.lsar_sweep(p_bar, cs[0], 1, want_diag="light", n=n)
wall = time.time() - t0
ph = diag["phases"].sum(0)
dev = float(np.sum(secs))
w = n - p_bar
print(f"C4 LSAR n={n} p_bar={p_bar} s={cs[0]}: device {dev:.2f} s (wall {wall:.2f}); "
      f"sample {ph[0]:.2f} s, solve {ph[1]:.2f} s, pass {ph[2]:.2f} s; "
      f"{p_bar * w / dev:.3e} rows*orders/s; p*={pstar}; methods {np.bincount(diag['method'])}")
sw = diag["svd_sweeps"]
print("SVD sweeps per lag: mean %.1f, max %d; by p: %s" % (sw[sw > 0].mean() if (sw > 0).any() else 0, sw.max(),
      [(p, int(sw[p - 1])) for p in (20, 50, 100, 200, 300, 400, 500) if p <= p_bar]))
fp64 = eng.probe_fp64_peak()
roof = sum(max(24.0 * w / 6537.3e9, (2.0 * p + 4.0) * w / (fp64 * 1e12)) for p in range(1, p_bar + 1))
print(f"pass roofline sum {roof:.2f} s (HBM 6537 GB/s, fp64 {fp64:.1f} TF/s) -> pass at {roof / ph[2] * 100:.0f} %")

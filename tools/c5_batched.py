"""BASELINE C5 through the batched sweep (tf_lsar_sweep_batch): 4096
independent series (n = 1e5, AR order 1..10, roots in [1.1, 3]), LSAR
p = 1..50, s = 2000, every lag one launch set for the whole batch.  Times
the batch (wall, includes H2D of the series and D2H of the results) and
checks a sample of fits against fit_many (the per-series path)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen
nser = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4096
rng = np.random.default_rng(2112)
pinned = "--pageable" not in sys.argv
if pinned:  # page-locked host buffer (as load_series_bin(pinned=True) gives): the upload runs at PCIe speed
    import torch
    Y = torch.empty((nser, 100_000), dtype=torch.float64, pin_memory=True).numpy()
else:
    Y = np.empty((nser, 100_000))
for k in range(nser):
    q = int(rng.integers(1, 11))
    Y[k] = gen.simulate_roots(gen.ar_roots(q, 1.1, 3.0, 1000 + k), 100_000, 1000 + k)
seeds = list(range(nser))
eng = tf.Engine(0)
tf.lsar_fit_batch(Y[:64], 50, 2000, seeds[:64], engine=eng)  # warm (allocations)
for rep in range(2):
    t0 = time.time()
    fits = tf.lsar_fit_batch(Y, 50, 2000, seeds, engine=eng)
    dt = time.time() - t0
    dev = sum(fits[0].per_lag_seconds) * nser  # per-fit seconds are the batch time / fits
    ro = nser * 50 * (100_000 - 50)
    print(f"C5 batched {nser} series ({'pinned' if pinned else 'pageable'} host series): {dt:.3f} s wall ({dev:.3f} s device lag loop), {ro / dt:.3e} rows*orders/s "
          f"(device {ro / dev:.3e}), {dt / nser * 1e3:.3f} ms/series", flush=True)
chk = list(range(0, nser, max(1, nser // 16)))
ref = tf.fit_many([Y[k] for k in chk], "lsar", 50, 2000, [seeds[k] for k in chk], workers=8)
agree = sum(1 for k, g in zip(chk, ref)
            if np.max(np.abs(np.array(fits[k].pacf.taus) - g.pacf.taus)) <= 1e-9 * np.max(np.abs(g.pacf.taus)))
same_p = sum(1 for k, g in zip(chk, ref) if fits[k].p_star == g.p_star)
print(f"check vs per-series path: {agree}/{len(chk)} fits with taus within 1e-9, {same_p}/{len(chk)} same p*")

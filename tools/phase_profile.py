"""Per-phase device-time breakdown of LSAR sweeps (development helper).
usage: python tools/phase_profile.py CONFIG C [n] [--ncu-range]"""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2112_12994_b200 as tf
from paper_2112_12994_b200 import gen

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
c = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else None
ncu_range = "--ncu-range" in sys.argv
y, _, p_bar, _ = gen.make_config_series(name, n=n)
eng = tf.Engine(0)
print("fp64 peak probe: %.2f TFLOP/s" % eng.probe_fp64_peak())
s = tf.TimeSeries(y)
fit = tf.lsar_fit(s, p_bar, c, 1, engine=eng, want_diag=True)  # warm
if ncu_range:
    import torch
    torch.cuda.profiler.start()
fit = tf.lsar_fit(s, p_bar, c, 2, engine=eng, want_diag=True)
if ncu_range:
    torch.cuda.profiler.stop()
ph = fit.diag["phases"]
tot = ph.sum()
print(f"{name} n={y.size} p_bar={p_bar} c={c}: total {tot*1e3:.2f} ms, launches {int(fit.diag['launches'][0])}")
for k, nm in enumerate(["sample", "solve", "pass"]):
    print(f"  {nm:7s} {ph[:, k].sum()*1e3:8.2f} ms  ({ph[:, k].sum()/tot*100:.1f}%)")
for p in [1, 2, 10, 50, 100, 150, 200]:
    if p <= p_bar:
        a, b, cc = ph[p - 1] * 1e6
        print(f"  p={p:3d}: sample {a:7.1f} us  solve {b:8.1f} us  pass {cc:7.1f} us  method {fit.diag['method'][p-1]}")
w = y.size - p_bar
bytes_pass = 40.0 * w
for p in [1, 50, 100, 200]:
    if p <= p_bar:
        t = ph[p - 1, 2]
        print(f"  pass p={p}: {bytes_pass/t/1e9:.0f} GB/s (40 B/row moved), {(2*p+4)*w/t/1e12:.2f} TFLOP/s")

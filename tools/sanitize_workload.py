"""Small workload touching every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): LSAR sweep (fused pass, draws, double-
double Gram, pivoted-Cholesky cluster, min-norm SVD cluster on a rank-deficient
C4-generator series), RH sweep (halving, sketch, CholeskyQR factor kernels,
Hankel row scores), the batched sweep (k_bsolve), exact / SRHT sweeps, the
LsarDriver step API, the FFT pass and the INT8 Gram (forced).  Usage: python tools/sanitize_workload.py"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2112_12994_b200 as tf  # noqa: E402
from paper_2112_12994_b200 import gen  # noqa: E402

eng = tf.Engine(0)
y = gen.simulate_roots(gen.ar_roots(6, 1.2, 3.0, 3), 12000, 3)
s = tf.TimeSeries(y)
f = tf.lsar_fit(s, 12, 600, 5, engine=eng)
r = tf.rh_fit(s, 12, 600, None, 5, engine=eng)
y4, _, _, _ = gen.make_config_series("C4", n=20000)
f4 = tf.lsar_fit(tf.TimeSeries(y4), 40, 800, 7, engine=eng, want_diag=True)
b = tf.lsar_fit_batch([y[:4000], y[4000:8000]], 6, 300, [1, 2], engine=eng)
e = tf.exact_fit(tf.TimeSeries(y[:3000]), 8, engine=eng)
h = tf.srht_fit(tf.TimeSeries(y[:3000]), 4, 300, 3, engine=eng)
d = tf.LsarDriver(s, 4, 300, 9, engine=eng)
st = d.advance(d.first_lag())
# the FFT pass (double-double spectra, TMA-staged spectrum) and the INT8
# tensor-core Gram (tcgen05 kind::i8), forced on at this small size
os.environ["TF_PASS"] = "fft"
os.environ["TF_GRAM"] = "i8"
eng2 = tf.Engine(0)
f5 = tf.lsar_fit(tf.TimeSeries(y4), 40, 800, 7, engine=eng2, want_diag=True)
print("sanitize workload ok:", f.p_star, r.p_star, f4.p_star, int(np.sum(f4.diag["method"])), b[0].p_star, e.p_star,
      h.p_star, st.p, f5.p_star)

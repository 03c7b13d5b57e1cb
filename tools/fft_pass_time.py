"""Per-lag pass time of the direct tensor-core FIR pass (TF_PASS=dmma) against
the FFT pass (TF_PASS=fft) on a C4-shaped sweep: one instrumented sweep per
mode (per-lag phase events), printed per lag band, plus the crossover lag.

  python tools/fft_pass_time.py [n] [p_bar] [c] [modes, e.g. "fft" or "dmma,fft"]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2112_12994_b200 as tf
    from paper_2112_12994_b200 import gen
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000_000
    p_bar = int(sys.argv[2]) if len(sys.argv) > 2 else 500
    c = int(sys.argv[3]) if len(sys.argv) > 3 else 200_000
    roots = gen.ar_roots(100, 1.05, 2.0, 2112_12994)
    res = {}
    modes = sys.argv[4].split(",") if len(sys.argv) > 4 else ["dmma", "fft"]
    for mode in modes:
        os.environ["TF_PASS"] = mode
        eng = tf.Engine(0)
        eng.generate_series(roots, n, 2112_12994, "normal")
        for w in range(2):
            out = eng.lsar_sweep(p_bar, c, 1, want_diag="light", n=n)
        a, b = eng.sweep_span(eng)
        ph = out[4]["phases"]
        res[mode] = dict(pass_s=ph[:, 2].tolist(), solve_s=float(ph[:, 1].sum()), sample_s=float(ph[:, 0].sum()),
                         sweep_s=(b - a) * 1e-3, taus=out[0].tolist(), p_star=out[3])
        eng.close()
        print(mode, "sweep %.3f s  pass %.3f  solve %.3f  sample %.3f  p* %d" % (
            res[mode]["sweep_s"], sum(res[mode]["pass_s"]), res[mode]["solve_s"], res[mode]["sample_s"], out[3]),
            flush=True)
    if len(modes) < 2:
        return
    d = np.array(res["dmma"]["pass_s"]) * 1e3
    f = np.array(res["fft"]["pass_s"]) * 1e3
    w = n - p_bar
    for lo in list(range(1, p_bar + 1, max(1, p_bar // 20))):
        hi = min(p_bar, lo + max(1, p_bar // 20) - 1)
        sl = slice(lo - 1, hi)
        print("lags %4d-%4d  dmma %8.3f ms  fft %8.3f ms  (fft %.1f B/row-equiv at 6544 GB/s: %.2f ms)" % (
            lo, hi, d[sl].mean(), f[sl].mean(), 42.7, 42.7 * w / 6544e9 * 1e3))
    cross = next((q for q in range(1, p_bar + 1) if f[q - 1:].max() <= d[q - 1:].min() or all(
        f[k] < d[k] for k in range(q - 1, p_bar))), None)
    best = np.minimum(d, f).sum() * 1e-3
    print("crossover lag (fft faster from here on):", cross, " pass with per-lag best: %.3f s" % best)
    tdiff = np.abs(np.array(res["fft"]["taus"]) - np.array(res["dmma"]["taus"])).max()
    print("max |tau_fft - tau_dmma| (RNG mode, draws may flip):", tdiff)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fft_pass_time.json"), "w") as fh:
        json.dump(dict(n=n, p_bar=p_bar, c=c, **{k: v for k, v in res.items()}), fh)


if __name__ == "__main__":
    main()
